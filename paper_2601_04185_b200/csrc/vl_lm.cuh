// CTA-cooperative fp64 passes over a point set: MSAC classification and the
// Levenberg-Marquardt / IRLS pose refinement.
//
//  * msac_pass  == posest._errors_sq + msac_score (posest.py:137-175): fp64,
//    behind-camera -> +inf error, cost sum w min(e2, tau^2), flags e2 < tau^2.
//    The per-point arithmetic is issued without FMA contraction in the
//    reference's operation order so flags agree bit-for-bit away from ties.
//  * lm_refine  == refine.refine_pose (refine.py:164-230) with TruncatedLoss
//    or CauchyLoss (:43-77), residuals (:90-100), analytic Jacobian
//    (:103-132), robust cost (:135-149), apply_delta (:80-87), and the exact
//    damping schedule.  One fused pass evaluates cost + gradient + the 21
//    unique entries of J^T W J at every candidate, so an accepted step
//    already carries the next iteration's normal equations (the reference
//    recomputes them at the same pose, so the values are identical).
//  Reductions are deterministic (fixed warp-shuffle tree + ordered warp sum).
//
// Point sets come in two layouts: the caller's AoS arrays (px (n,2), X (n,3),
// w (n)) and the packed layout the library writes for data it re-reads many
// times (scoring subset, compacted inliers): three double2 per point,
// (X, Y), (Z, u), (v, w) — three coalesced 16-byte loads per point.
#pragma once
#include "vl_common.cuh"

namespace vl {

enum LossKind { kTruncated = 0, kCauchy = 1 };
constexpr int kRed = 28;  // cost, g[6], H upper triangle [21]

struct AosPts {
  const double* px;
  const double* X;
  const double* w;
  int n;
  __device__ __forceinline__ void load(int i, double* P, double& u, double& v, double& ww) const {
    P[0] = X[3 * i];
    P[1] = X[3 * i + 1];
    P[2] = X[3 * i + 2];
    u = px[2 * i];
    v = px[2 * i + 1];
    ww = w[i];
  }
};

struct PackedPts {
  const double2* p;  // [3n]
  int n;
  __device__ __forceinline__ void load(int i, double* P, double& u, double& v, double& ww) const {
    const double2 a = __ldg(p + 3 * i), b = __ldg(p + 3 * i + 1), c = __ldg(p + 3 * i + 2);
    P[0] = a.x;
    P[1] = a.y;
    P[2] = b.x;
    u = b.y;
    v = c.x;
    ww = c.y;
  }
};

__device__ __forceinline__ void pack_point(double2* dst, int i, const double* P, double u, double v, double w) {
  dst[3 * i] = make_double2(P[0], P[1]);
  dst[3 * i + 1] = make_double2(P[2], u);
  dst[3 * i + 2] = make_double2(v, w);
}

template <int NT>
struct LMShared {
  double R[9], t[3];
  Pose cur, cand;
  double red[kRed + 2];
  double red2[kRed + 2];
  double scratch[(NT / 32) * (kRed + 2)];
  double A[36], b[6];
  int flag;
  int ibuf[NT / 32];
  long long cnt[16];
};

// ---------------------------------------------------------------- clusters
// A query may be processed by a thread-block cluster (up to 8 CTAs on 8
// SMs): every pass splits the points over the cluster, CTA partial sums are
// combined through distributed shared memory in fixed rank order (so every
// CTA holds bit-identical totals), and the LM control flow runs redundantly
// in every CTA.  With a 1-CTA launch these are no-ops.
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned n;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  return n;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ double cl_load(const double* local_smem, unsigned rank) {
  unsigned addr = (unsigned)__cvta_generic_to_shared(local_smem), raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(addr), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(raddr) : "memory");
  return v;
}
__device__ __forceinline__ long long cl_load_ll(const long long* local_smem, unsigned rank) {
  unsigned addr = (unsigned)__cvta_generic_to_shared(local_smem), raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(addr), "r"(rank));
  long long v;
  asm volatile("ld.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(raddr) : "memory");
  return v;
}

// sm.red[0..K) holds this CTA's block totals; replace them by the cluster
// totals (sum over ranks 0..n-1 in order).  Call from all threads.
template <int NT, int K>
__device__ __forceinline__ void cluster_total(LMShared<NT>& sm) {
  const unsigned n = cl_size();
  if (n == 1) return;
  cl_sync();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (unsigned r = 0; r < n; ++r) s += cl_load(&sm.red[threadIdx.x], r);
    sm.red2[threadIdx.x] = s;
  }
  cl_sync();  // every rank has read every partial before anyone overwrites sm.red
  if (threadIdx.x < K) sm.red[threadIdx.x] = sm.red2[threadIdx.x];
  __syncthreads();
}

// Packed points streamed through a shared-memory ring by TMA bulk copies
// (cp.async.bulk global -> shared, mbarrier completion): the LM / MSAC
// passes over the scoring subset and the compacted inliers re-read the same
// 48-B records every pass, and the plain loads left the passes latency bound
// (ncu: long_scoreboard 35 % of the k_scan stalls).  Each CTA walks its
// contiguous share of the points in chunks of kStageCh records; chunk c lands
// in ring slot c % kStageN while the CTA works on the earlier slots.  Within
// a CTA, thread t still visits points t, t + NT, t + 2 NT, ... in order, so a
// 1-CTA launch accumulates exactly as the unstaged loop does.
constexpr int kStageCh = 512;  // records per chunk (24 KB)
#ifndef VL_STAGE_N
#define VL_STAGE_N 3
#endif
constexpr int kStageN = VL_STAGE_N;  // ring depth
constexpr size_t kStageBytes = (size_t)kStageN * kStageCh * 3 * sizeof(double2);

struct StagedPts {
  const double2* p;  // [3n] global
  int n;
  double2* ring;     // dynamic smem [kStageN][3 * kStageCh]
  uint64_t* bar;     // smem mbarriers [kStageN]
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void stage_issue(const StagedPts& ps, int lo, int cnt, int c) {
  const int slot = c % kStageN;
  const int m = min(kStageCh, cnt - c * kStageCh);
  const unsigned bytes = (unsigned)m * 48u;
  const unsigned bar = smem_u32(ps.bar + slot);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(ps.ring + (size_t)slot * 3 * kStageCh)), "l"(ps.p + 3 * (int64_t)(lo + c * kStageCh)),
               "r"(bytes), "r"(bar)
               : "memory");
}

// Invalidate the ring's mbarriers once every thread is past its last wait, so
// the next pass's mbarrier.init does not act on a live barrier.
__device__ __forceinline__ void stage_inval(uint64_t* bars) {
  __syncthreads();
  if (threadIdx.x == 0)
    for (int b = 0; b < kStageN; ++b)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bars + b)) : "memory");
  __syncthreads();
}

__device__ __forceinline__ void stage_wait(const StagedPts& ps, int c) {
  const unsigned bar = smem_u32(ps.bar + c % kStageN);
  const unsigned parity = (unsigned)(c / kStageN) & 1u;
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// fn(P, u, v, w) for every point of this CTA's share (cluster rank r owns
// [n r / cs, n (r+1) / cs)); all threads of the CTA must call it.
template <int NT, typename F>
__device__ __forceinline__ void staged_for_each(const StagedPts& ps, F&& fn) {
  const int r = (int)cl_rank(), cs = (int)cl_size();
  const int lo = (int)((int64_t)ps.n * r / cs), hi = (int)((int64_t)ps.n * (r + 1) / cs);
  const int cnt = hi - lo;
  const int nch = (cnt + kStageCh - 1) / kStageCh;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kStageN; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ps.bar + b)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int c = 0; c < min(kStageN, nch); ++c) stage_issue(ps, lo, cnt, c);
  for (int c = 0; c < nch; ++c) {
    stage_wait(ps, c);
    const double2* buf = ps.ring + (size_t)(c % kStageN) * 3 * kStageCh;
    const int m = min(kStageCh, cnt - c * kStageCh);
    for (int i = threadIdx.x; i < m; i += NT) {
      const double2 a = buf[3 * i], b = buf[3 * i + 1], cc = buf[3 * i + 2];
      const double P[3] = {a.x, a.y, b.x};
      fn(P, b.y, cc.x, cc.y);
    }
    __syncthreads();  // every thread is done with the slot before it is refilled
    if (threadIdx.x == 0 && c + kStageN < nch) stage_issue(ps, lo, cnt, c + kStageN);
  }
  stage_inval(ps.bar);  // the next pass re-initialises them
}

template <typename PS>
struct is_staged {
  static constexpr bool value = false;
};
template <>
struct is_staged<StagedPts> {
  static constexpr bool value = true;
};

// Load rotation matrix + translation of `p` into shared memory (thread 0).
template <int NT>
__device__ __forceinline__ void set_eval_pose(LMShared<NT>& sm, const Pose& p) {
  if (threadIdx.x == 0) {
    q2R(p.q, sm.R);
    sm.t[0] = p.t[0];
    sm.t[1] = p.t[1];
    sm.t[2] = p.t[2];
  }
  __syncthreads();
}

__device__ __forceinline__ void cam_point(const double* R, const double* t, const double* X,
                                          double& x, double& y, double& z) {
  // X @ R.T + t, no contraction
  x = dadd(dadd(dadd(dmul(X[0], R[0]), dmul(X[1], R[1])), dmul(X[2], R[2])), t[0]);
  y = dadd(dadd(dadd(dmul(X[0], R[3]), dmul(X[1], R[4])), dmul(X[2], R[5])), t[1]);
  z = dadd(dadd(dadd(dmul(X[0], R[6]), dmul(X[1], R[7])), dmul(X[2], R[8])), t[2]);
}

// fp64 MSAC error of one point (posest._errors_sq order); +inf behind camera.
__device__ __forceinline__ double msac_e2(const double* R, const double* t, const Intr& in, const double* P,
                                          double u, double v) {
  double x, y, z;
  cam_point(R, t, P, x, y, z);
  const bool front = z > 0;
  const double zs = front ? z : 1.0;
  // (fx x) / zs via one reciprocal + remainder correction: the correctly
  // rounded quotient except for rare double-rounding ties (1 ulp), which can
  // only move a flag for e2 within ~1e-16 relative of tau^2 (the parity bar
  // already excludes |e - tau| < 1e-6 px)
  const double iz = __drcp_rn(zs);
  const double ax = dmul(in.fx, x), ay = dmul(in.fy, y);
  const double qx = ax * iz, qy = ay * iz;
  double du = fma(fma(-qx, zs, ax), iz, qx);
  du = dadd(du, dsub(in.cx, u));
  double dv = fma(fma(-qy, zs, ay), iz, qy);
  dv = dadd(dv, dsub(in.cy, v));
  double e2 = dmul(du, du);
  e2 = dadd(e2, dmul(dv, dv));
  return front ? e2 : CUDART_INF;
}

// MSAC pass with the pose currently in sm.R / sm.t.  Writes flags (if not
// null), returns cost and inlier count in sm.red[0], sm.red[1].
template <int NT, typename PS>
__device__ void msac_pass(LMShared<NT>& sm, const PS& ps, const Intr& in, double tau, uint8_t* flags) {
  const double t2 = dmul(tau, tau);
  double R[9], t[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = sm.R[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = sm.t[k];
  double acc[2] = {0.0, 0.0};
  if constexpr (is_staged<PS>::value) {
    staged_for_each<NT>(ps, [&](const double* P0, double u0, double v0, double w0) {
      const double e0 = msac_e2(R, t, in, P0, u0, v0);
      acc[0] = acc[0] + dmul(w0, fmin(e0, t2));
      acc[1] += e0 < t2 ? 1.0 : 0.0;
    });
    block_sum<NT, 2>(acc, sm.scratch, sm.red);
    cluster_total<NT, 2>(sm);
    return;
  } else {
  const int step = NT * (int)cl_size();
  int i = threadIdx.x + NT * (int)cl_rank();
  // four points per trip: all loads in flight before the arithmetic (the
  // full-set passes stream 48 B per point from HBM); accumulation stays in
  // point order, so the sums equal the one-point loop's
  constexpr int U = 4;
  for (; i + (U - 1) * step < ps.n; i += U * step) {
    double P[U][3], u[U], v[U], w[U];
#pragma unroll
    for (int k = 0; k < U; ++k) ps.load(i + k * step, P[k], u[k], v[k], w[k]);
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const double e = msac_e2(R, t, in, P[k], u[k], v[k]);
      acc[0] = acc[0] + dmul(w[k], fmin(e, t2));
      acc[1] += e < t2 ? 1.0 : 0.0;
      if (flags) flags[i + k * step] = e < t2 ? 1 : 0;
    }
  }
  for (; i < ps.n; i += step) {
    double P0[3], u0, v0, w0;
    ps.load(i, P0, u0, v0, w0);
    const double e0 = msac_e2(R, t, in, P0, u0, v0);
    acc[0] = acc[0] + dmul(w0, fmin(e0, t2));
    acc[1] += e0 < t2 ? 1.0 : 0.0;
    if (flags) flags[i] = e0 < t2 ? 1 : 0;
  }
  block_sum<NT, 2>(acc, sm.scratch, sm.red);
  cluster_total<NT, 2>(sm);
  }
}

// Cost / gradient / normal-matrix contribution of one point.
template <bool GRAD>
__device__ __forceinline__ void lm_point(const double* R, const double* t, const Intr& in, int kind, double s2,
                                         const double* P, double u_obs, double v_obs, double w, double* acc,
                                         double& behind) {
  // camera point with FMAs (3 per row instead of 3 mul + 3 add): the LM
  // cost only steers the schedule; classification keeps msac_pass's
  // reference-order arithmetic
  const double x = fma(P[2], R[2], fma(P[1], R[1], fma(P[0], R[0], t[0])));
  const double y = fma(P[2], R[5], fma(P[1], R[4], fma(P[0], R[3], t[1])));
  const double z = fma(P[2], R[8], fma(P[1], R[7], fma(P[0], R[6], t[2])));
  if (!(z > 0)) {
    behind = 1.0;
    if (kind == kTruncated) acc[0] += dmul(w, s2);
    return;
  }
  // (fx x) / z and (fy y) / z from one correctly rounded reciprocal plus a
  // remainder correction (the quotient is correctly rounded but for rare
  // double-rounding ties; the LM cost only steers the schedule — classification
  // flags come from msac_pass's exact divisions)
  const double iz = __drcp_rn(z);
  const double ax = dmul(in.fx, x), ay = dmul(in.fy, y);
  const double qx = ax * iz, qy = ay * iz;
  const double u = dadd(fma(fma(-qx, z, ax), iz, qx), in.cx);
  const double v = dadd(fma(fma(-qy, z, ay), iz, qy), in.cy);
  const double ru = dsub(u, u_obs);
  const double rv = dsub(v, v_obs);
  const double e2 = dadd(dmul(ru, ru), dmul(rv, rv));
  double rho, wt;
  if (kind == kTruncated) {
    rho = fmin(e2, s2);
    wt = (e2 < s2) ? 1.0 : 0.0;
  } else {
    // Cauchy (refine.py:69-77): r = e2 / s2, rho = s2/2 log1p(r), w = 1/2 / (1 + r);
    // the two quotients from correctly rounded reciprocals (<= 1 ulp)
    const double r = dmul(e2, __drcp_rn(s2));
    rho = dmul(dmul(0.5, s2), log1p(r));
    wt = dmul(0.5, __drcp_rn(dadd(1.0, r)));
  }
  acc[0] += dmul(w, rho);
  if (GRAD) {
    const double wr = dmul(w, wt);
    if (wr != 0.0) {
      // dpi/dX_cam (refine.py:115-118) from one reciprocal: the normal
      // equations only steer the step (the cost above keeps the reference's
      // exact divisions), so 1 ulp here changes nothing the schedule compares
      const double p00 = in.fx * iz, p02 = -(in.fx * x) * (iz * iz);
      const double p11 = in.fy * iz, p12 = -(in.fy * y) * (iz * iz);
      double J0[6], J1[6];
      J0[0] = p02 * y;
      J0[1] = p00 * z + p02 * (-x);
      J0[2] = p00 * (-y);
      J0[3] = p00;
      J0[4] = 0.0;
      J0[5] = p02;
      J1[0] = p11 * (-z) + p12 * y;
      J1[1] = p12 * (-x);
      J1[2] = p11 * x;
      J1[3] = 0.0;
      J1[4] = p11;
      J1[5] = p12;
      // weighted rows once, then g += Jw^T r and H += Jw^T J: 2 FMA per entry.
      // J0[4] = J1[3] = 0 exactly, so every product with one of them is an
      // exact zero: those entries keep only their other term, as a rounded
      // product added to the accumulator — the bits the two-term expression
      // gives (fma(x, y, +-0) = round(x y); fma(0, y, p) = p) — and H[3][4]
      // stays 0.  Same results, 16 fewer fp64 operations per point.
      double W0[6], W1[6];
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        W0[a] = a == 4 ? 0.0 : wr * J0[a];
        W1[a] = a == 3 ? 0.0 : wr * J1[a];
      }
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        if (a == 3) acc[1 + a] += dmul(W0[a], ru);
        else if (a == 4) acc[1 + a] += dmul(W1[a], rv);
        else acc[1 + a] += W0[a] * ru + W1[a] * rv;
      }
      int k = 7;
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = a; b < 6; ++b, ++k) {
          const bool z0 = a == 4 || b == 4, z1 = a == 3 || b == 3;
          if (z0 && z1) continue;  // H[3][4]: both terms exactly zero
          if (z0) acc[k] += dmul(W1[a], J1[b]);
          else if (z1) acc[k] += dmul(W0[a], J0[b]);
          else acc[k] += W0[a] * J0[b] + W1[a] * J1[b];
        }
    }
  }
}

// Fused robust-cost (+ gradient + normal matrix) pass at the pose in sm.R/t.
// Result: sm.red[0] = cost (inf for Cauchy with a point behind the camera),
// sm.red[1..6] = g (without the factor 2), sm.red[7..27] = H upper (no 2).
template <int NT, bool GRAD, typename PS>
__device__ void lm_pass(LMShared<NT>& sm, const PS& ps, const Intr& in, int kind, double scale) {
  const double s2 = dmul(scale, scale);
  double R[9], t[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = sm.R[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = sm.t[k];
  double acc[kRed];
#pragma unroll
  for (int k = 0; k < kRed; ++k) acc[k] = 0.0;
  double behind = 0.0;
  if constexpr (is_staged<PS>::value) {
    staged_for_each<NT>(ps, [&](const double* P0, double u0, double v0, double w0) {
      lm_point<GRAD>(R, t, in, kind, s2, P0, u0, v0, w0, acc, behind);
    });
  } else {
    const int step = NT * (int)cl_size();
    int i = threadIdx.x + NT * (int)cl_rank();
    for (; i + step < ps.n; i += 2 * step) {
      double P0[3], u0, v0, w0, P1[3], u1, v1, w1;
      ps.load(i, P0, u0, v0, w0);
      ps.load(i + step, P1, u1, v1, w1);
      lm_point<GRAD>(R, t, in, kind, s2, P0, u0, v0, w0, acc, behind);
      lm_point<GRAD>(R, t, in, kind, s2, P1, u1, v1, w1, acc, behind);
    }
    if (i < ps.n) {
      double P0[3], u0, v0, w0;
      ps.load(i, P0, u0, v0, w0);
      lm_point<GRAD>(R, t, in, kind, s2, P0, u0, v0, w0, acc, behind);
    }
  }
  // slot kRed carries the behind-camera count (a deterministic OR)
  if (GRAD) {
    double a[kRed + 1];
#pragma unroll
    for (int k = 0; k < kRed; ++k) a[k] = acc[k];
    a[kRed] = behind;
    block_sum<NT, kRed + 1>(a, sm.scratch, sm.red);
    cluster_total<NT, kRed + 1>(sm);
  } else {
    double a1[2] = {acc[0], behind};
    block_sum<NT, 2>(a1, sm.scratch, sm.red);
    cluster_total<NT, 2>(sm);
    if (threadIdx.x == 0) sm.red[kRed] = sm.red[1];
    __syncthreads();
  }
  if (kind == kCauchy && sm.red[kRed] != 0.0) {
    __syncthreads();
    if (threadIdx.x == 0) sm.red[0] = CUDART_INF;
  }
  __syncthreads();
}

// 6x6 LU with partial pivoting in shared memory (np.linalg.solve / LAPACK
// gesv semantics: fails only on an exactly zero pivot).  One thread.
// 6x6 solve with partial pivoting (the damped normal equations), on one
// thread.  The matrix is copied into registers and the elimination fully
// unrolled — every index static, pivot row swaps as predicated selects — so
// the serial section the other warps wait for is register latency, not ~200
// dependent shared-memory round trips (ncu: that barrier was 15.6 % of the C5
// k_scan stall samples).  Same operations in the same order as the smem
// version, hence the same bits.
__device__ __noinline__ bool solve6_smem(double* As, double* bs) {
  double A[36], b[6];
#pragma unroll
  for (int i = 0; i < 36; ++i) A[i] = As[i];
#pragma unroll
  for (int i = 0; i < 6; ++i) b[i] = bs[i];
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    int p = k;
    double pv = fabs(A[6 * k + k]);
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      const double v = fabs(A[6 * i + k]);
      if (v > pv) {
        pv = v;
        p = i;
      }
    }
    double piv = A[6 * k + k];
#pragma unroll
    for (int i = k + 1; i < 6; ++i) piv = p == i ? A[6 * i + k] : piv;
    if (piv == 0.0) ok = false;
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      if (p == i) {
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const double tmp = A[6 * k + j];
          A[6 * k + j] = A[6 * i + j];
          A[6 * i + j] = tmp;
        }
        const double tb = b[k];
        b[k] = b[i];
        b[i] = tb;
      }
    }
    const double inv = A[6 * k + k];
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      const double f = A[6 * i + k] / inv;
#pragma unroll
      for (int j = k + 1; j < 6; ++j) A[6 * i + j] -= f * A[6 * k + j];
      b[i] -= f * b[k];
    }
  }
  if (!ok) return false;
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double s = b[i];
#pragma unroll
    for (int j = i + 1; j < 6; ++j) s -= A[6 * i + j] * b[j];
    b[i] = s / A[6 * i + i];
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) bs[i] = b[i];
  return true;
}

struct LMResult {
  int converged;
  int iterations;
  double cost;
};

// Levenberg-Marquardt refinement of `start` (all threads pass the same
// value).  Result pose in sm.cur.  trace (global, optional): accepted costs.
// g and the upper triangle of H live in shared memory (sm.red after each
// pass); every thread keeps only the scalars of the schedule.
template <int NT, typename PS>
__device__ LMResult lm_refine(LMShared<NT>& sm, const PS& ps, const Intr& in, const Pose& start, int kind,
                              double scale, int max_iters, double gtol, double ctol, double* trace,
                              int* trace_len) {
  __shared__ double gH[kRed];
  if (threadIdx.x == 0) sm.cur = start;
  __syncthreads();
  set_eval_pose(sm, sm.cur);
  lm_pass<NT, true>(sm, ps, in, kind, scale);
  double cost = sm.red[0];
  if (threadIdx.x < kRed) gH[threadIdx.x] = 2.0 * sm.red[threadIdx.x];
  int ntr = 0;
  if (trace && threadIdx.x == 0) trace[0] = cost;
  ntr = 1;
  double lam = 1e-6;
  int conv = 0;
  int it = 0;
  __syncthreads();
  for (it = 1; it <= max_iters; ++it) {
    double gn = 0.0;
#pragma unroll
    for (int a = 0; a < 6; ++a) gn += gH[1 + a] * gH[1 + a];
    if (sqrt(gn) < gtol) {
      conv = 1;
      break;
    }
    bool accepted = false;
    double cc = 0.0;
    for (int trial = 0; trial < 25; ++trial) {
      if (threadIdx.x == 0) {
        int k = 7;
        for (int a = 0; a < 6; ++a)
          for (int b = a; b < 6; ++b, ++k) {
            sm.A[6 * a + b] = gH[k];
            sm.A[6 * b + a] = gH[k];
          }
        k = 7;
        for (int a = 0; a < 6; ++a) {
          const double dga = fmax(gH[k], 1e-12);  // diag(H) entry
          sm.A[7 * a] = sm.A[7 * a] + lam * dga;
          sm.b[a] = -gH[1 + a];
          k += 6 - a;
        }
        const bool ok = solve6_smem(sm.A, sm.b);
        sm.flag = ok ? 1 : 0;
        if (ok) {
          apply_delta(sm.cur, sm.b, sm.cand);
          q2R(sm.cand.q, sm.R);
          sm.t[0] = sm.cand.t[0];
          sm.t[1] = sm.cand.t[1];
          sm.t[2] = sm.cand.t[2];
        }
      }
      __syncthreads();
      if (!sm.flag) {
        lam *= 10.0;
        __syncthreads();
        continue;
      }
      lm_pass<NT, true>(sm, ps, in, kind, scale);
      cc = sm.red[0];
      if (cc <= cost) {
        accepted = true;
        break;
      }
      lam *= 10.0;
      if (lam > 1e14) break;
    }
    if (!accepted) break;
    lam = fmax(lam / 3.0, 1e-12);
    const double drop = cost - cc;
    cost = cc;
    __syncthreads();
    if (threadIdx.x < kRed) gH[threadIdx.x] = 2.0 * sm.red[threadIdx.x];
    if (threadIdx.x == 0) {
      sm.cur = sm.cand;
      if (trace) trace[ntr] = cost;
    }
    ++ntr;
    __syncthreads();
    if (drop < ctol * fmax(cost, 1e-300)) {
      conv = 1;
      break;
    }
  }
  if (it > max_iters) it = max_iters;
  if (trace_len && threadIdx.x == 0) *trace_len = ntr;
  LMResult r;
  r.converged = conv;
  r.iterations = it;
  r.cost = cost;
  return r;
}

}  // namespace vl
