// Shared device helpers: pose algebra (fp64), block reductions, constants.
//
// Pose algebra mirrors pkg/src/visloc/geometry.py: quat_multiply :79-89,
// quat_to_matrix :92-100, matrix_to_quat (Shepperd) :103-127,
// rotvec_to_quat :130-141, Pose.__post_init__ canonicalisation :160-171.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

#ifndef VL_HD
#define VL_HD __host__ __device__ __forceinline__
#ifndef VL_P3P_NOINLINE
#define VL_P3P_NOINLINE 0  // measured: noinline solver stages make k_p3p 28 % slower (C3 10.3 -> 13.2 ms)
#endif
#if VL_P3P_NOINLINE
#define VL_HD_BIG __host__ __device__ __noinline__  // large solver stages: one copy of the code (i-cache)
#else
#define VL_HD_BIG VL_HD
#endif
#endif

namespace vl {

constexpr int kMaxSolPerSample = 4;

struct Intr {
  double fx, fy, cx, cy;
};

// Camera-from-world pose as stored by the reference: unit quaternion (w>=0) + t.
struct Pose {
  double q[4];
  double t[3];
};

// Point set in the reference's AoS layout: px (n,2), X (n,3), w (n).
struct PointSet {
  const double* px;
  const double* X;
  const double* w;
  int n;
};

VL_HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
VL_HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
VL_HD double dsub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}

VL_HD void qmul(const double* a, const double* b, double* o) {
  const double aw = a[0], ax = a[1], ay = a[2], az = a[3];
  const double bw = b[0], bx = b[1], by = b[2], bz = b[3];
  o[0] = dsub(dsub(dsub(dmul(aw, bw), dmul(ax, bx)), dmul(ay, by)), dmul(az, bz));
  o[1] = dsub(dadd(dadd(dmul(aw, bx), dmul(ax, bw)), dmul(ay, bz)), dmul(az, by));
  o[2] = dadd(dadd(dsub(dmul(aw, by), dmul(ax, bz)), dmul(ay, bw)), dmul(az, bx));
  o[3] = dadd(dsub(dadd(dmul(aw, bz), dmul(ax, by)), dmul(ay, bx)), dmul(az, bw));
}

VL_HD void q2R(const double* q, double* R) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(z, z))));
  R[1] = dmul(2.0, dsub(dmul(x, y), dmul(w, z)));
  R[2] = dmul(2.0, dadd(dmul(x, z), dmul(w, y)));
  R[3] = dmul(2.0, dadd(dmul(x, y), dmul(w, z)));
  R[4] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(z, z))));
  R[5] = dmul(2.0, dsub(dmul(y, z), dmul(w, x)));
  R[6] = dmul(2.0, dsub(dmul(x, z), dmul(w, y)));
  R[7] = dmul(2.0, dadd(dmul(y, z), dmul(w, x)));
  R[8] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y))));
}

VL_HD double norm4(const double* q) {
  return sqrt(dadd(dadd(dadd(dmul(q[0], q[0]), dmul(q[1], q[1])), dmul(q[2], q[2])), dmul(q[3], q[3])));
}

// Pose.__post_init__: renormalise only when |n-1| > 1e-12, then w >= 0.
VL_HD void canon(double* q) {
  const double n = norm4(q);
  if (fabs(n - 1.0) > 1e-12) {
    for (int i = 0; i < 4; ++i) q[i] = q[i] / n;
  }
  if (q[0] < 0) {
    for (int i = 0; i < 4; ++i) q[i] = -q[i];
  }
}

// Shepperd's method, branch order of geometry.py:103-127, then q / ||q||.
VL_HD void R2q(const double* R, double* q) {
  const double tr = dadd(dadd(R[0], R[4]), R[8]);
  double s;
  if (tr > 0) {
    s = sqrt(dadd(tr, 1.0)) * 2.0;
    q[0] = 0.25 * s;
    q[1] = dsub(R[7], R[5]) / s;
    q[2] = dsub(R[2], R[6]) / s;
    q[3] = dsub(R[3], R[1]) / s;
  } else if (R[0] >= R[4] && R[0] >= R[8]) {
    s = sqrt(dsub(dsub(dadd(1.0, R[0]), R[4]), R[8])) * 2.0;
    q[0] = dsub(R[7], R[5]) / s;
    q[1] = 0.25 * s;
    q[2] = dadd(R[1], R[3]) / s;
    q[3] = dadd(R[2], R[6]) / s;
  } else if (R[4] >= R[8]) {
    s = sqrt(dsub(dsub(dadd(1.0, R[4]), R[0]), R[8])) * 2.0;
    q[0] = dsub(R[2], R[6]) / s;
    q[1] = dadd(R[1], R[3]) / s;
    q[2] = 0.25 * s;
    q[3] = dadd(R[5], R[7]) / s;
  } else {
    s = sqrt(dsub(dsub(dadd(1.0, R[8]), R[0]), R[4])) * 2.0;
    q[0] = dsub(R[3], R[1]) / s;
    q[1] = dadd(R[2], R[6]) / s;
    q[2] = dadd(R[5], R[7]) / s;
    q[3] = 0.25 * s;
  }
  const double n = norm4(q);
  for (int i = 0; i < 4; ++i) q[i] = q[i] / n;
}

VL_HD void rotvec2q(const double* w, double* q) {
  const double th = sqrt(dadd(dadd(dmul(w[0], w[0]), dmul(w[1], w[1])), dmul(w[2], w[2])));
  if (th < 1e-12) {
    const double h = 0.5 * th;
    q[0] = 1.0 - dmul(h, h) / 2.0;
    q[1] = 0.5 * w[0];
    q[2] = 0.5 * w[1];
    q[3] = 0.5 * w[2];
    const double n = norm4(q);
    for (int i = 0; i < 4; ++i) q[i] = q[i] / n;
    return;
  }
  const double s = sin(0.5 * th);
  q[0] = cos(0.5 * th);
  q[1] = dmul(w[0] / th, s);
  q[2] = dmul(w[1] / th, s);
  q[3] = dmul(w[2] / th, s);
}

// Pose.from_rt (geometry.py:174-176): quaternion round trip + canonicalisation.
VL_HD void pose_from_Rt(const double* R, const double* t, Pose& p) {
  R2q(R, p.q);
  canon(p.q);
  p.t[0] = t[0];
  p.t[1] = t[1];
  p.t[2] = t[2];
}

// refine.apply_delta (refine.py:80-87): left-compose (omega, nu).
VL_HD void apply_delta(const Pose& in, const double* d, Pose& out) {
  double dq[4], qn[4], Rd[9];
  rotvec2q(d, dq);
  qmul(dq, in.q, qn);
  double dqc[4] = {dq[0], dq[1], dq[2], dq[3]};
  canon(dqc);
  q2R(dqc, Rd);
  for (int i = 0; i < 3; ++i) {
    const double r = dadd(dadd(dmul(Rd[3 * i], in.t[0]), dmul(Rd[3 * i + 1], in.t[1])),
                          dmul(Rd[3 * i + 2], in.t[2]));
    out.t[i] = dadd(r, d[3 + i]);
  }
  canon(qn);
  for (int i = 0; i < 4; ++i) out.q[i] = qn[i];
}

// ---------------------------------------------------------------- reductions
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_min_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum of K doubles per thread (fixed tree order).
// `scratch` must hold (NT/32)*K doubles; result broadcast into out[K] (shared).
template <int NT, int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* scratch, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) scratch[wid * K + k] = v[k];
  }
  __syncthreads();
  constexpr int NW = NT / 32;
  for (int k = threadIdx.x; k < K; k += NT) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += scratch[w * K + k];
    out[k] = s;
  }
  __syncthreads();
}

}  // namespace vl
