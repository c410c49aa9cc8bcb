// Depth lifting: confidence gate + depth decode/fetch + unproject + world
// transform + order-preserving compaction, for many (query, entry,
// direction) field segments in one launch sequence.
//
// Reference: localizer.lift (localizer.py:134-197), interp_depth_many
// (:87-115), matchio.filter_matches_arrays (matchio.py:203-218) and
// mapstore.dequantize_depth (mapstore.py:122-134; applied here through a
// per-map code -> f32 table built with the reference formula).
//
// Output order is the reference's: segments in the caller's order (entry id,
// then db->query before query->db), cells row-major inside a segment.
// Three kernels: per-block keep counts -> one-CTA exclusive scan over blocks
// -> recompute + block-local scan + write.  HBM-bound: every kept match is
// written once (px 2 f64, X 3 f64, w f64, entry i32 = 52 B).
#include <climits>
#include <cuda_fp16.h>
#include "vl_common.cuh"
#include "vl_lift.h"

namespace vl {

constexpr int kLiftThreads = 256;
constexpr int kLiftPerThread = 8;
constexpr int kLiftBlockCells = kLiftThreads * kLiftPerThread;  // 2048

__device__ __forceinline__ float depth_value(const LiftDepth& D, int64_t idx, bool& valid) {
  switch (D.kind) {
    case kDepthF32:
      valid = D.valid[idx] != 0;
      return ((const float*)D.values)[idx];
    case kDepthF16:
      valid = D.valid[idx] != 0;
      return __half2float(((const __half*)D.values)[idx]);
    case kDepthCode8: {
      const int c = ((const uint8_t*)D.values)[idx];
      valid = c > 0;
      return D.lut[c];
    }
    default: {
      const int c = ((const uint16_t*)D.values)[idx];
      valid = c > 0;
      return D.lut[c];
    }
  }
}

// Bilinear depth with the all-4-valid rule (localizer.py:87-115).  Returns ok.
__device__ __forceinline__ bool interp_depth(const LiftDepth& D, double px, double py, double& d) {
  const int w = D.w, h = D.h;
  const double x = dsub(px, 0.5), y = dsub(py, 0.5);
  const bool inside = (x >= 0) && (x <= (double)(w - 1)) && (y >= 0) && (y <= (double)(h - 1));
  double xf = floor(x), yf = floor(y);
  xf = fmin(fmax(xf, 0.0), (double)(w - 2));
  yf = fmin(fmax(yf, 0.0), (double)(h - 2));
  const int x0 = (int)xf, y0 = (int)yf;
  const double fx = fmin(fmax(dsub(x, (double)x0), 0.0), 1.0);
  const double fy = fmin(fmax(dsub(y, (double)y0), 0.0), 1.0);
  if (!inside) return false;
  bool v00, v10, v01, v11;
  const int64_t r0 = (int64_t)y0 * w, r1 = (int64_t)(y0 + 1) * w;
  const double d00 = depth_value(D, r0 + x0, v00);
  const double d10 = depth_value(D, r0 + x0 + 1, v10);
  const double d01 = depth_value(D, r1 + x0, v01);
  const double d11 = depth_value(D, r1 + x0 + 1, v11);
  if (!(v00 && v10 && v01 && v11)) return false;
  const double gx = dsub(1.0, fx), gy = dsub(1.0, fy);
  double s = dmul(dmul(d00, gx), gy);
  s = dadd(s, dmul(dmul(d10, fx), gy));
  s = dadd(s, dmul(dmul(d01, gx), fy));
  s = dadd(s, dmul(dmul(d11, fx), fy));
  d = s;
  return true;
}

// world point (xc - t) @ R for pixel (u, v) at depth d in the db camera
__device__ __forceinline__ void lift_point(const LiftDepth& D, double u, double v, double d, double* X) {
  const double xc0 = dmul(__ddiv_rn(dsub(u, D.cx), D.fx), d);
  const double xc1 = dmul(__ddiv_rn(dsub(v, D.cy), D.fy), d);
  const double v0 = dsub(xc0, D.t[0]), v1 = dsub(xc1, D.t[1]), v2 = dsub(d, D.t[2]);
#pragma unroll
  for (int j = 0; j < 3; ++j) X[j] = dadd(dadd(dmul(v0, D.R[j]), dmul(v1, D.R[3 + j])), dmul(v2, D.R[6 + j]));
}

template <typename T>
struct CellResult {
  bool keep;
  double px[2];
  double X[3];
  double w;
};

// Evaluate one cell.  mode 0: lift (keep = gate && depth ok); mode 1: gate only
// (px = source, X[0..1] = target, X[2] = flat cell index).
template <typename T>
__device__ __forceinline__ bool cell_eval(const LiftSeg& S, const LiftDepth* depths, int cell, T thr, int mode,
                                          CellResult<T>& r) {
  const T* conf = (const T*)S.confidence;
  const T c = conf[cell];
  // gate (matchio.py:211): (conf >= thr) & (conf > 0), compared in the field dtype
  if (!((c >= thr) && (c > (T)0))) return false;
  const int row = cell / S.gw, col = cell - row * S.gw;
  const T* tg = (const T*)S.targets;
  const double tx = (double)tg[2 * (int64_t)cell], ty = (double)tg[2 * (int64_t)cell + 1];
  const double sx = dmul((double)col + 0.5, S.scale_x), sy = dmul((double)row + 0.5, S.scale_y);
  r.w = (double)c;
  if (mode == 1) {
    r.px[0] = sx;
    r.px[1] = sy;
    r.X[0] = tx;
    r.X[1] = ty;
    r.X[2] = (double)cell;
    return true;
  }
  const LiftDepth& D = depths[S.depth];
  double d;
  if (S.direction == 0) {
    // db -> query: direct lookup at the db cell (localizer.py:164-168)
    double fxi = floor(dmul(sx, D.sx_depth)), fyi = floor(dmul(sy, D.sy_depth));
    const int ix = (int)fmin(fmax(fxi, 0.0), (double)(D.w - 1));
    const int iy = (int)fmin(fmax(fyi, 0.0), (double)(D.h - 1));
    bool ok;
    d = (double)depth_value(D, (int64_t)iy * D.w + ix, ok);
    if (!ok) return false;
    lift_point(D, sx, sy, d, r.X);
    r.px[0] = tx;
    r.px[1] = ty;
  } else {
    // query -> db: bilinear at the subpixel target (localizer.py:181-196)
    if (!interp_depth(D, dmul(tx, D.sx_depth), dmul(ty, D.sy_depth), d)) return false;
    lift_point(D, tx, ty, d, r.X);
    r.px[0] = sx;
    r.px[1] = sy;
  }
  return true;
}

__device__ __forceinline__ int find_seg(const int64_t* seg_blk0, int nseg, int64_t b) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg_blk0[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <typename T>
__global__ void __launch_bounds__(kLiftThreads) k_lift_count(LiftArgs a, int mode) {
  const int64_t b = blockIdx.x;
  const int s = find_seg(a.seg_blk0, a.nseg, b);
  const LiftSeg S = a.segs[s];
  const int cells = S.gw * S.gh;
  const int base = (int)(b - a.seg_blk0[s]) * kLiftBlockCells + threadIdx.x * kLiftPerThread;
  int cnt = 0;
  for (int i = 0; i < kLiftPerThread; ++i) {
    const int cell = base + i;
    if (cell >= cells) break;
    CellResult<T> r;
    cnt += cell_eval<T>(S, a.depths, cell, (T)a.threshold, mode, r) ? 1 : 0;
  }
  __shared__ int wsum[kLiftThreads / 32];
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kLiftThreads / 32; ++w) t += wsum[w];
    a.blk_count[b] = t;
  }
}

// One CTA: exclusive scan of block counts, segment offsets, total.
__global__ void __launch_bounds__(1024) k_lift_scan(LiftArgs a) {
  __shared__ int64_t wtot[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < a.nblk; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < a.nblk ? a.blk_count[i] : 0;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wtot[wid] = x;
    __syncthreads();
    int64_t wb = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      if (w < wid) wb += wtot[w];
      tot += wtot[w];
    }
    if (i < a.nblk) a.blk_off[i] = carry + wb + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  for (int s = threadIdx.x; s < a.nseg; s += 1024) a.seg_off[s] = a.blk_off[a.seg_blk0[s]];
  if (threadIdx.x == 0) a.seg_off[a.nseg] = carry;
}

template <typename T>
__global__ void __launch_bounds__(kLiftThreads) k_lift_write(LiftArgs a, int mode) {
  __shared__ int wtot[kLiftThreads / 32];
  const int64_t b = blockIdx.x;
  const int s = find_seg(a.seg_blk0, a.nseg, b);
  const LiftSeg S = a.segs[s];
  const int cells = S.gw * S.gh;
  const int base = (int)(b - a.seg_blk0[s]) * kLiftBlockCells + threadIdx.x * kLiftPerThread;
  CellResult<T> r[kLiftPerThread];
  unsigned keep = 0;
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < kLiftPerThread; ++i) {
    const int cell = base + i;
    if (cell < cells && cell_eval<T>(S, a.depths, cell, (T)a.threshold, mode, r[i])) {
      keep |= 1u << i;
      ++cnt;
    }
  }
  // block-local exclusive scan (row-major order preserved)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wtot[wid] = x;
  __syncthreads();
  int wb = 0;
  for (int w = 0; w < wid; ++w) wb += wtot[w];
  int64_t pos = a.blk_off[b] + wb + x - cnt;
#pragma unroll
  for (int i = 0; i < kLiftPerThread; ++i) {
    if (!(keep >> i & 1u)) continue;
    if (pos < a.capacity) {
      a.px_out[2 * pos] = r[i].px[0];
      a.px_out[2 * pos + 1] = r[i].px[1];
      a.X_out[3 * pos] = r[i].X[0];
      a.X_out[3 * pos + 1] = r[i].X[1];
      a.X_out[3 * pos + 2] = r[i].X[2];
      a.w_out[pos] = r[i].w;
      if (a.entry_out) a.entry_out[pos] = S.entry;
    }
    ++pos;
  }
}

int launch_lift(const LiftArgs& a, int field_f64, int mode, cudaStream_t st) {
  if (a.nblk <= 0) return 0;
  if (field_f64) k_lift_count<double><<<(unsigned)a.nblk, kLiftThreads, 0, st>>>(a, mode);
  else k_lift_count<float><<<(unsigned)a.nblk, kLiftThreads, 0, st>>>(a, mode);
  k_lift_scan<<<1, 1024, 0, st>>>(a);
  return 2;
}

int launch_lift_write(const LiftArgs& a, int field_f64, int mode, cudaStream_t st) {
  if (a.nblk <= 0) return 0;
  if (field_f64) k_lift_write<double><<<(unsigned)a.nblk, kLiftThreads, 0, st>>>(a, mode);
  else k_lift_write<float><<<(unsigned)a.nblk, kLiftThreads, 0, st>>>(a, mode);
  return 1;
}

int lift_block_cells() { return kLiftBlockCells; }

// Standalone bilinear interpolation (interp_depth_many, localizer.py:87-115).
__global__ void k_interp(LiftDepth D, const double* pts, int n, double* vals, uint8_t* ok) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  const bool o = interp_depth(D, pts[2 * i], pts[2 * i + 1], d);
  vals[i] = o ? d : 0.0;
  ok[i] = o ? 1 : 0;
}

int launch_interp(const LiftDepth& D, const double* pts, int n, double* vals, uint8_t* ok, cudaStream_t st) {
  if (n <= 0) return 0;
  k_interp<<<(n + 255) / 256, 256, 0, st>>>(D, pts, n, vals, ok);
  return 1;
}

// Standalone decode (dequantize_depth, mapstore.py:122-134): codes -> f32 + valid.
__global__ void k_decode(LiftDepth D, int64_t n, float* vals, uint8_t* valid) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool v;
  const float d = depth_value(D, i, v);
  vals[i] = v ? d : 0.f;
  valid[i] = v ? 1 : 0;
}

int launch_decode(const LiftDepth& D, int64_t n, float* vals, uint8_t* valid, cudaStream_t st) {
  if (n <= 0) return 0;
  k_decode<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(D, n, vals, valid);
  return 1;
}

}  // namespace vl
