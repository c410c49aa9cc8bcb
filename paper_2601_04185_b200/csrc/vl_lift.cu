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
// Three kernels: per-block keep counts (+ IMLC content validation) -> one-CTA
// exclusive scan over blocks -> recompute + block-local ordered scan + write.
// HBM-bound: every kept match is written once (px 2 f64, X 3 f64, w f64,
// entry i32 = 52 B).  Fields are read either as planar arrays or straight
// from IMLC records (12 B/cell, matchio.py:9-20) — in HBM or in mapped pinned
// host memory.
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

struct CellResult {
  double px[2];
  double X[3];
  double w;
};

// One field cell: confidence + target, in the field's own dtype for the gate.
template <typename T>
struct CellIn {
  T c;
  double tx, ty;
};

template <typename T>
__device__ __forceinline__ CellIn<T> load_cell(const LiftSeg& S, int cell) {
  CellIn<T> in;
  if (S.layout == kLayoutImlc) {
    // IMLC record (x f32, y f32, conf f32), matchio.py:18-19
    const float* r = (const float*)S.targets + 3 * (int64_t)cell;
    in.c = (T)r[2];
    in.tx = (double)r[0];
    in.ty = (double)r[1];
  } else {
    const T* tg = (const T*)S.targets;
    in.c = ((const T*)S.confidence)[cell];
    in.tx = (double)tg[2 * (int64_t)cell];
    in.ty = (double)tg[2 * (int64_t)cell + 1];
  }
  return in;
}

// gate (matchio.py:211): (conf >= thr) & (conf > 0), compared in the field
// dtype (IMLC records are f32: T = float is exact for them)
template <typename T>
__device__ __forceinline__ bool gate(T c, T thr) {
  return (c >= thr) && (c > (T)0);
}

__device__ __forceinline__ void source_px(const LiftSeg& S, int cell, double& sx, double& sy) {
  const int row = cell / S.gw, col = cell - row * S.gw;
  sx = dmul((double)col + 0.5, S.scale_x);
  sy = dmul((double)row + 0.5, S.scale_y);
}

__device__ __forceinline__ void direct_tap(const LiftDepth& D, double sx, double sy, int64_t& idx) {
  const double fxi = floor(dmul(sx, D.sx_depth)), fyi = floor(dmul(sy, D.sy_depth));
  const int ix = (int)fmin(fmax(fxi, 0.0), (double)(D.w - 1));
  const int iy = (int)fmin(fmax(fyi, 0.0), (double)(D.h - 1));
  idx = (int64_t)iy * D.w + ix;
}

// Evaluate one gated cell.  mode 0: lift (false when the depth is invalid);
// mode 1: gate only (px = source, X[0..1] = target, X[2] = flat cell index).
template <typename T>
__device__ __forceinline__ bool cell_eval(const LiftSeg& S, const LiftDepth* depths, int cell, const CellIn<T>& in,
                                          int mode, CellResult& r) {
  double sx, sy;
  source_px(S, cell, sx, sy);
  r.w = (double)in.c;
  if (mode == 1) {
    r.px[0] = sx;
    r.px[1] = sy;
    r.X[0] = in.tx;
    r.X[1] = in.ty;
    r.X[2] = (double)cell;
    return true;
  }
  const LiftDepth& D = depths[S.depth];
  double d;
  if (S.direction == 0) {
    // db -> query: direct lookup at the db cell (localizer.py:164-168)
    int64_t idx;
    direct_tap(D, sx, sy, idx);
    bool ok;
    d = (double)depth_value(D, idx, ok);
    if (!ok) return false;
    lift_point(D, sx, sy, d, r.X);
    r.px[0] = in.tx;
    r.px[1] = in.ty;
  } else {
    // query -> db: bilinear at the subpixel target (localizer.py:181-196)
    if (!interp_depth(D, dmul(in.tx, D.sx_depth), dmul(in.ty, D.sy_depth), d)) return false;
    lift_point(D, in.tx, in.ty, d, r.X);
    r.px[0] = sx;
    r.px[1] = sy;
  }
  return true;
}

// Keep decision only (count pass): gate + depth validity, no lift arithmetic.
template <typename T>
__device__ __forceinline__ bool cell_keep(const LiftSeg& S, const LiftDepth* depths, int cell, const CellIn<T>& in,
                                          int mode) {
  if (mode == 1) return true;
  const LiftDepth& D = depths[S.depth];
  double sx, sy;
  if (S.direction == 0) {
    source_px(S, cell, sx, sy);
    int64_t idx;
    direct_tap(D, sx, sy, idx);
    bool ok;
    (void)depth_value(D, idx, ok);
    return ok;
  }
  double d;
  return interp_depth(D, dmul(in.tx, D.sx_depth), dmul(in.ty, D.sy_depth), d);
}

// IMLC content rules of CorrespondenceField.__post_init__ (matchio.py:99-109)
__device__ __forceinline__ int content_flags(float c, double tx, double ty) {
  int f = 0;
  if (!(isfinite(c) && c >= 0.f && c <= 1.f)) f |= kFieldBadConf;
  if (c > 0.f && !(isfinite(tx) && isfinite(ty))) f |= kFieldBadTarget;
  return f;
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

// A block covers kLiftBlockCells consecutive cells of one segment; warp w owns
// the contiguous run [w*256, (w+1)*256) of them and iteration i handles cells
// w*256 + i*32 + lane, so every load and output store of a warp touches
// consecutive addresses and the write pass can rank cells inside each warp
// with no block barrier (per-warp counts come from this pass).
#ifndef VL_LIFT_CMINB
#define VL_LIFT_CMINB 8  // min resident CTAs of the count pass (register cap; 8 measured best)
#endif
#ifndef VL_LIFT_WMINB
#define VL_LIFT_WMINB 5  // same for the write pass (5 measured best; small spills cost less than the occupancy)
#endif
constexpr int kLiftWarps = kLiftThreads / 32;
constexpr int kLiftWarpCells = kLiftBlockCells / kLiftWarps;  // 256

template <typename T>
__global__ void __launch_bounds__(kLiftThreads, VL_LIFT_CMINB) k_lift_count(LiftArgs a, int mode) {
  const int64_t b = blockIdx.x;
  const int s = find_seg(a.seg_blk0, a.nseg, b);
  const LiftSeg S = a.segs[s];
  const int cells = S.gw * S.gh;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cw = (int)(b - a.seg_blk0[s]) * kLiftBlockCells + wid * kLiftWarpCells;
  const T thr = (T)a.threshold;
  int cnt = 0, flags = 0;
#pragma unroll 4
  for (int i = 0; i < kLiftPerThread; ++i) {
    const int cell = cw + i * 32 + lane;
    if (cell < cells) {
      const CellIn<T> in = load_cell<T>(S, cell);
      if (S.layout == kLayoutImlc) flags |= content_flags((float)in.c, in.tx, in.ty);
      if (gate<T>(in.c, thr) && cell_keep<T>(S, a.depths, cell, in, mode)) ++cnt;
    }
  }
  __shared__ int wsum[kLiftWarps];
  __shared__ int wflag[kLiftWarps];
  cnt = warp_sum(cnt);
  flags = __reduce_or_sync(0xffffffffu, (unsigned)flags);
  if (lane == 0) {
    wsum[wid] = cnt;
    wflag[wid] = flags;
    a.warp_count[b * kLiftWarps + wid] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0, f = 0;
    for (int w = 0; w < kLiftWarps; ++w) {
      t += wsum[w];
      f |= wflag[w];
    }
    a.blk_count[b] = t;
    if (f && a.seg_flags) atomicOr(a.seg_flags + s, f);
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
  for (int s = threadIdx.x; s < a.nseg; s += 1024) {
    const int64_t o = a.blk_off[a.seg_blk0[s]];
    a.seg_off[s] = o;
    if (a.seg_off_host) a.seg_off_host[s] = o;
    if (a.seg_flags_host) a.seg_flags_host[s] = a.seg_flags ? a.seg_flags[s] : 0;
  }
  if (threadIdx.x == 0) {
    a.seg_off[a.nseg] = carry;
    if (a.seg_off_host) a.seg_off_host[a.nseg] = carry;
  }
}

__global__ void k_lift_prep(uint64_t* dst, const uint64_t* src, int64_t words, int* zero, int zero_n) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = i0; i < words; i += step) dst[i] = src[i];
  for (int64_t i = i0; i < zero_n; i += step) zero[i] = 0;
}

int launch_lift_prep(void* dst, const void* src_host, size_t bytes, int* zero, int zero_n, cudaStream_t st) {
  const int64_t words = (int64_t)(bytes / 8);
  const int64_t n = words > zero_n ? words : zero_n;
  const int blocks = (int)((n + 255) / 256 < 148 ? (n + 255) / 256 : 148);
  k_lift_prep<<<blocks > 0 ? blocks : 1, 256, 0, st>>>((uint64_t*)dst, (const uint64_t*)src_host, words, zero, zero_n);
  return 1;
}

template <typename T>
__global__ void __launch_bounds__(kLiftThreads, VL_LIFT_WMINB) k_lift_write(LiftArgs a, int mode) {
  const int64_t b = blockIdx.x;
  const int s = find_seg(a.seg_blk0, a.nseg, b);
  const LiftSeg S = a.segs[s];
  const int cells = S.gw * S.gh;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cw = (int)(b - a.seg_blk0[s]) * kLiftBlockCells + wid * kLiftWarpCells;
  if (cw >= cells) return;  // whole warp past the segment end
  const T thr = (T)a.threshold;
  const unsigned lt = (1u << lane) - 1u;
  // this warp's first output row: block offset + the block's earlier warps
  int64_t pos = a.blk_off[b];
  {
    const int c = lane < wid ? a.warp_count[b * kLiftWarps + lane] : 0;
    pos += warp_sum(c);
  }
  // X rows (24 B) of the warp's kept cells are staged in shared memory and
  // stored as one contiguous run of doubles (3 fully coalesced stores per
  // iteration instead of three 8-B stores at a 24-B stride)
  __shared__ double sX[kLiftWarps][3 * 32];
  double* xs = sX[wid];
  for (int i = 0; i < kLiftPerThread; ++i) {
    const int cell = cw + i * 32 + lane;
    if (cw + i * 32 >= cells) break;  // uniform across the warp
    CellResult r;
    bool keep = false;
    if (cell < cells) {
      const CellIn<T> in = load_cell<T>(S, cell);
      keep = gate<T>(in.c, thr) && cell_eval<T>(S, a.depths, cell, in, mode, r);
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    const int nk = __popc(m);
    if (keep) {
      const int k = __popc(m & lt);
      const int64_t p = pos + k;
      xs[3 * k] = r.X[0];
      xs[3 * k + 1] = r.X[1];
      xs[3 * k + 2] = r.X[2];
      if (p < a.capacity) {
        reinterpret_cast<double2*>(a.px_out)[p] = make_double2(r.px[0], r.px[1]);
        a.w_out[p] = r.w;
        if (a.entry_out) a.entry_out[p] = S.entry;
      }
    }
    __syncwarp();
    const int64_t lim = 3 * (a.capacity - pos);  // doubles of X_out still inside the capacity
    for (int j = lane; j < 3 * nk; j += 32)
      if (j < lim) a.X_out[3 * pos + j] = xs[j];
    __syncwarp();
    pos += nk;
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
