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
#include <cstdlib>
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

// Block-uniform parameters of a segment and of its depth map, held in
// registers for the whole block (loaded once with uniform __ldg: the
// generic-pointer struct copies of the first version went through local
// memory and cost an LD per use).
struct SegP {
  int gw, cells, entry, direction, layout, depth;
  double scale_x, scale_y;
  const void* targets;
  const void* conf;
};

struct DepP {
  int w, h;
  double wm1, hm1, wm2, hm2;  // w - 1, h - 1, w - 2, h - 2 as doubles (clamp bounds)
  const void* values;
  const uint8_t* valid;
  const float* lut;
  double fx, fy, cx, cy, sxd, syd;
};

__device__ __forceinline__ SegP load_seg(const LiftSeg* g) {
  SegP S;
  S.gw = __ldg(&g->gw);
  S.cells = S.gw * __ldg(&g->gh);
  S.entry = __ldg(&g->entry);
  S.direction = __ldg(&g->direction);
  S.layout = __ldg(&g->layout);
  S.depth = __ldg(&g->depth);
  S.scale_x = __ldg(&g->scale_x);
  S.scale_y = __ldg(&g->scale_y);
  S.targets = (const void*)__ldg((const unsigned long long*)&g->targets);
  S.conf = (const void*)__ldg((const unsigned long long*)&g->confidence);
  return S;
}

__device__ __forceinline__ DepP load_dep(const LiftDepth* g) {
  DepP D;
  D.w = __ldg(&g->w);
  D.h = __ldg(&g->h);
  D.wm1 = (double)(D.w - 1);
  D.hm1 = (double)(D.h - 1);
  D.wm2 = (double)(D.w - 2);
  D.hm2 = (double)(D.h - 2);
  D.values = (const void*)__ldg((const unsigned long long*)&g->values);
  D.valid = (const uint8_t*)__ldg((const unsigned long long*)&g->valid);
  D.lut = (const float*)__ldg((const unsigned long long*)&g->lut);
  D.fx = __ldg(&g->fx);
  D.fy = __ldg(&g->fy);
  D.cx = __ldg(&g->cx);
  D.cy = __ldg(&g->cy);
  D.sxd = __ldg(&g->sx_depth);
  D.syd = __ldg(&g->sy_depth);
  return D;
}

// Depth taps per stored kind (kind is a template parameter: the inner loops
// carry no switch).  tap_ok: validity only (count pass: no value / LUT load).
template <int KIND>
__device__ __forceinline__ bool tap_ok(const DepP& D, int idx) {
  if (KIND == kDepthF32 || KIND == kDepthF16) return __ldg(D.valid + idx) != 0;
  if (KIND == kDepthCode8) return __ldg((const uint8_t*)D.values + idx) != 0;
  return __ldg((const uint16_t*)D.values + idx) != 0;
}

template <int KIND>
__device__ __forceinline__ float tap_val(const DepP& D, int idx, bool& ok) {
  if (KIND == kDepthF32) {
    ok = __ldg(D.valid + idx) != 0;
    return __ldg((const float*)D.values + idx);
  }
  if (KIND == kDepthF16) {
    ok = __ldg(D.valid + idx) != 0;
    return __half2float(__ldg((const __half*)D.values + idx));
  }
  const int c = KIND == kDepthCode8 ? (int)__ldg((const uint8_t*)D.values + idx)
                                    : (int)__ldg((const uint16_t*)D.values + idx);
  ok = c > 0;
  return __ldg(D.lut + c);
}

// Bilinear sample position (localizer.py:97-105): clamped base tap and
// fractions, `inside` = the reference's inside test.
struct Bilin {
  int i00;
  double fx, fy;
  bool inside;
};

__device__ __forceinline__ Bilin bilin(const DepP& D, double px, double py) {
  const double x = dsub(px, 0.5), y = dsub(py, 0.5);
  Bilin b;
  b.inside = (x >= 0) && (x <= D.wm1) && (y >= 0) && (y <= D.hm1);
  // x0 = clip(floor(x), 0, w - 2) kept as a double: x - x0 needs no int -> double conversion
  const double xf = fmin(fmax(floor(x), 0.0), D.wm2);
  const double yf = fmin(fmax(floor(y), 0.0), D.hm2);
  b.fx = fmin(fmax(dsub(x, xf), 0.0), 1.0);
  b.fy = fmin(fmax(dsub(y, yf), 0.0), 1.0);
  b.i00 = (int)yf * D.w + (int)xf;
  return b;
}

template <int KIND>
__device__ __forceinline__ bool interp_ok(const DepP& D, double px, double py) {
  const Bilin b = bilin(D, px, py);
  if (!b.inside) return false;
  return tap_ok<KIND>(D, b.i00) && tap_ok<KIND>(D, b.i00 + 1) && tap_ok<KIND>(D, b.i00 + D.w) &&
         tap_ok<KIND>(D, b.i00 + D.w + 1);
}

// value: d00(1-fx)(1-fy) + d10 fx(1-fy) + d01(1-fx)fy + d11 fx fy, left to right (localizer.py:106-112)
template <int KIND>
__device__ __forceinline__ bool interp_val(const DepP& D, double px, double py, double& d) {
  const Bilin b = bilin(D, px, py);
  if (!b.inside) return false;
  bool v00, v10, v01, v11;
  const double d00 = tap_val<KIND>(D, b.i00, v00);
  const double d10 = tap_val<KIND>(D, b.i00 + 1, v10);
  const double d01 = tap_val<KIND>(D, b.i00 + D.w, v01);
  const double d11 = tap_val<KIND>(D, b.i00 + D.w + 1, v11);
  if (!(v00 && v10 && v01 && v11)) return false;
  const double gx = dsub(1.0, b.fx), gy = dsub(1.0, b.fy);
  double s = dmul(dmul(d00, gx), gy);
  s = dadd(s, dmul(dmul(d10, b.fx), gy));
  s = dadd(s, dmul(dmul(d01, gx), b.fy));
  s = dadd(s, dmul(dmul(d11, b.fx), b.fy));
  d = s;
  return true;
}

// db -> query direct lookup index: int(src * depth/image) clipped (localizer.py:164-165)
__device__ __forceinline__ int direct_idx(const DepP& D, double sx, double sy) {
  const double fxi = floor(dmul(sx, D.sxd)), fyi = floor(dmul(sy, D.syd));
  const int ix = (int)fmin(fmax(fxi, 0.0), D.wm1);
  const int iy = (int)fmin(fmax(fyi, 0.0), D.hm1);
  return iy * D.w + ix;
}

// world point (xc - t) @ R for pixel (u, v) at depth d in the db camera
__device__ __forceinline__ void lift_point(const DepP& D, const double* R, const double* t, double u, double v,
                                           double d, double* X) {
  const double xc0 = dmul(__ddiv_rn(dsub(u, D.cx), D.fx), d);
  const double xc1 = dmul(__ddiv_rn(dsub(v, D.cy), D.fy), d);
  const double v0 = dsub(xc0, t[0]), v1 = dsub(xc1, t[1]), v2 = dsub(d, t[2]);
#pragma unroll
  for (int j = 0; j < 3; ++j) X[j] = dadd(dadd(dmul(v0, R[j]), dmul(v1, R[3 + j])), dmul(v2, R[6 + j]));
}

// One field cell in the field's own dtype (IMLC records are f32).  `srec`:
// the block's records staged in shared memory (cell c0 first), or null.
template <typename T>
__device__ __forceinline__ void load_cell(const SegP& S, int cell, T& c, double& tx, double& ty,
                                          const float* srec = nullptr, int c0 = 0) {
  if (srec) {
    const float* r = srec + 3 * (cell - c0);
    c = (T)r[2];
    tx = (double)r[0];
    ty = (double)r[1];
  } else if (S.layout == kLayoutImlc) {
    // IMLC record (x f32, y f32, conf f32), matchio.py:18-19
    const float* r = (const float*)S.targets + 3 * (int64_t)cell;
    c = (T)__ldg(r + 2);
    tx = (double)__ldg(r);
    ty = (double)__ldg(r + 1);
  } else {
    const T* tg = (const T*)S.targets;
    c = __ldg((const T*)S.conf + cell);
    tx = (double)__ldg(tg + 2 * (int64_t)cell);
    ty = (double)__ldg(tg + 2 * (int64_t)cell + 1);
  }
}

// gate (matchio.py:211): (conf >= thr) & (conf > 0), compared in the field
// dtype (IMLC records are f32: T = float is exact for them)
template <typename T>
__device__ __forceinline__ bool gate(T c, T thr) {
  return (c >= thr) && (c > (T)0);
}

// IMLC content rules of CorrespondenceField.__post_init__ (matchio.py:99-109)
__device__ __forceinline__ int content_flags(float c, double tx, double ty) {
  int f = 0;
  if (!(isfinite(c) && c >= 0.f && c <= 1.f)) f |= kFieldBadConf;
  if (c > 0.f && !(isfinite(tx) && isfinite(ty))) f |= kFieldBadTarget;
  return f;
}

// Source pixel of a cell: ((col + 0.5) sx, (row + 0.5) sy) (matchio.py:215-216)
__device__ __forceinline__ void source_px(const SegP& S, int row, int col, double& sx, double& sy) {
  sx = dmul((double)col + 0.5, S.scale_x);
  sy = dmul((double)row + 0.5, S.scale_y);
}

// Lane's (row, col) walk: cell advances by 32 per iteration.
struct CellWalk {
  int cell, row, col;
  __device__ __forceinline__ CellWalk(int c0, int gw) : cell(c0), row(c0 / gw), col(c0 - (c0 / gw) * gw) {}
  __device__ __forceinline__ void next(int gw) {
    cell += 32;
    col += 32;
    while (col >= gw) {
      col -= gw;
      ++row;
    }
  }
  // grids at least 32 cells wide wrap at most once per step: no loop
  __device__ __forceinline__ void next_wide(int gw) {
    cell += 32;
    col += 32;
    const bool wrap = col >= gw;
    col -= wrap ? gw : 0;
    row += wrap ? 1 : 0;
  }
};

// KIND = kGateOnly: mode 1 (gate only, no depth)
constexpr int kGateOnly = 4;

// db -> query segments: the depth tap and the normalised ray of a cell
// depend only on its column and row (localizer.py:164-176), so a block
// computes them once per column / row — the same fp64 operations, cached —
// instead of once per cell: ix = clip(int(sx * dw / W)), xn = (sx - cx) / fx
// (the division), likewise for rows.  Used when the grid is at most
// kTabCols wide and the block spans at most kTabRows rows.
constexpr int kTabCols = 512, kTabRows = 72;

struct Dir0Tab {
  const int* ix;       // [gw]
  const int* iy;       // [rows of the block], row0 first
  const double* xn;    // [gw]  (write pass)
  const double* yn;    // [rows]
  int row0;
  bool on;             // tables filled (else the per-cell path)
};

// All threads call it; the caller's next __syncthreads publishes the tables.
// Returns false (tables unused) when the segment does not qualify.
__device__ __forceinline__ bool fill_dir0_tab(const SegP& S, const DepP& D, int c0, bool with_n, int* ix, int* iy,
                                              double* xn, double* yn, Dir0Tab& tab) {
  const int row0 = c0 / S.gw, row1 = (min(S.cells, c0 + kLiftBlockCells) - 1) / S.gw;
  tab.on = false;
  if (S.direction != 0 || S.gw > kTabCols || row1 - row0 + 1 > kTabRows) return false;
  for (int col = threadIdx.x; col < S.gw; col += blockDim.x) {
    const double sx = dmul((double)col + 0.5, S.scale_x);
    ix[col] = (int)fmin(fmax(floor(dmul(sx, D.sxd)), 0.0), (double)(D.w - 1));
    if (with_n) xn[col] = __ddiv_rn(dsub(sx, D.cx), D.fx);
  }
  for (int r = threadIdx.x; r <= row1 - row0; r += blockDim.x) {
    const double sy = dmul((double)(row0 + r) + 0.5, S.scale_y);
    iy[r] = (int)fmin(fmax(floor(dmul(sy, D.syd)), 0.0), (double)(D.h - 1));
    if (with_n) yn[r] = __ddiv_rn(dsub(sy, D.cy), D.fy);
  }
  tab.ix = ix;
  tab.iy = iy;
  tab.xn = xn;
  tab.yn = yn;
  tab.row0 = row0;
  tab.on = true;
  return true;
}

// world point from the normalised ray (xn, yn) at depth d: identical to
// lift_point's arithmetic with the quotients precomputed
__device__ __forceinline__ void lift_point_n(const double* R, const double* t, double xn, double yn, double d,
                                             double* X) {
  const double xc0 = dmul(xn, d), xc1 = dmul(yn, d);
  const double v0 = dsub(xc0, t[0]), v1 = dsub(xc1, t[1]), v2 = dsub(d, t[2]);
#pragma unroll
  for (int j = 0; j < 3; ++j) X[j] = dadd(dadd(dmul(v0, R[j]), dmul(v1, R[3 + j])), dmul(v2, R[6 + j]));
}

// The block's 2048 IMLC records (24 KB, 12 B each) are pulled into shared
// memory by ONE bulk async copy (cp.async.bulk, TMA engine, mbarrier
// completion) instead of 3 dependent 4-B loads per lane per iteration: the
// count pass was latency bound (ncu: 1.8 TB/s, 22 % of DRAM peak, IPC 2.3).
// Records of a 16-B aligned segment start 16-B aligned for every block
// (2048 x 12 B = 24576 B); a sub-16-B tail of the last block is copied by
// plain loads.  Returns srec, or null (planar fields / unaligned records:
// the global path).  Every thread of the block must call it; it ends with a
// block barrier on both paths.
__device__ __forceinline__ unsigned lift_smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ const float* stage_records(const SegP& S, int c0, float* srec, uint64_t* bar) {
  if (S.layout != kLayoutImlc || (reinterpret_cast<uintptr_t>(S.targets) & 15) || c0 >= S.cells) {
    __syncthreads();  // block-uniform: callers rely on this barrier either way
    return nullptr;
  }
  const int ncell = min(kLiftBlockCells, S.cells - c0);
  const float* src = (const float*)S.targets + 3 * (int64_t)c0;
  const unsigned bytes = (unsigned)ncell * 12u, bulk = bytes & ~15u;
  const unsigned b = lift_smem_u32(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bulk) : "memory");
    if (bulk)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(lift_smem_u32(srec)), "l"(src), "r"(bulk), "r"(b) : "memory");
  }
  for (unsigned k = bulk / 4 + threadIdx.x; k < bytes / 4; k += blockDim.x) srec[k] = __ldg(src + k);
  __syncthreads();  // barrier initialised, tail stored
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LIFT_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra LIFT_WAIT_%=;\n}" ::"r"(b)
      : "memory");
  return srec;
}


// A block covers kLiftBlockCells consecutive cells of one segment; warp w owns
// the contiguous run [w*256, (w+1)*256) of them and iteration i handles cells
// w*256 + i*32 + lane, so every load and output store of a warp touches
// consecutive addresses and the write pass can rank cells inside each warp
// with no block barrier (per-warp counts come from this pass).
#ifndef VL_LIFT_CMINB
#define VL_LIFT_CMINB 6  // min resident CTAs of the count pass (40 registers: no spills)
#endif
#ifndef VL_LIFT_WMINB
#define VL_LIFT_WMINB 5  // same for the write pass
#endif
constexpr int kLiftWarps = kLiftThreads / 32;
constexpr int kLiftWarpCells = kLiftBlockCells / kLiftWarps;  // 256

// A block covers kLiftBlockCells consecutive cells of one segment; warp w owns
// the contiguous run [w*256, (w+1)*256) of them and iteration i handles cells
// w*256 + i*32 + lane, so every load and output store of a warp touches
// consecutive addresses and the write pass can rank cells inside each warp
// with no block barrier (per-warp counts come from the count pass).
template <typename T, int DIR, int KIND>
__device__ __forceinline__ int count_run(const SegP& S, const DepP& D, T thr, int cw, int lane, int& flags,
                                         const float* srec, int c0, const Dir0Tab tab) {
  int cnt = 0;
  CellWalk cwk(cw + lane, S.gw);
#pragma unroll 2
  for (int i = 0; i < kLiftPerThread; ++i, cwk.next(S.gw)) {
    if (cwk.cell >= S.cells) break;
    T c;
    double tx, ty;
    load_cell<T>(S, cwk.cell, c, tx, ty, srec, c0);
    if (S.layout == kLayoutImlc) flags |= content_flags((float)c, tx, ty);
    bool keep = gate<T>(c, thr);
    if (keep && KIND != kGateOnly) {
      if (DIR == 0) {
        if (tab.on) {
          keep = tap_ok<KIND>(D, tab.iy[cwk.row - tab.row0] * D.w + tab.ix[cwk.col]);
        } else {
          double sx, sy;
          source_px(S, cwk.row, cwk.col, sx, sy);
          keep = tap_ok<KIND>(D, direct_idx(D, sx, sy));
        }
      } else {
        keep = interp_ok<KIND>(D, dmul(tx, D.sxd), dmul(ty, D.syd));
      }
    }
    cnt += keep ? 1 : 0;
  }
  return cnt;
}

// Count of a warp's run from the block's staged IMLC records (f32), in
// groups of kCountGroup cells: first every cell of the group is gated and
// validated and its depth-tap index formed (shared memory and ALU only),
// then the group's tap loads are issued back to back with no branch in
// between (a cell that failed the gate reads tap 0 and is not counted), so a
// lane has kCountGroup (db -> query) or 4 x kCountGroup (query -> db) loads
// in flight instead of one dependent load per cell (count_run: ncu r02s,
// long_scoreboard the top stall, 2.5 TB/s).  Same decisions as count_run.
constexpr int kCountGroup = 4;

__device__ __forceinline__ int content_flags_f(float c, float tx, float ty) {
  int f = 0;
  if (!(c >= 0.f && c <= 1.f)) f |= kFieldBadConf;  // false for NaN and +-inf: isfinite implied
  if (c > 0.f && !(isfinite(tx) && isfinite(ty))) f |= kFieldBadTarget;
  return f;
}

template <int DIR, int KIND>
__device__ __forceinline__ int count_run_staged(const SegP& S, const DepP& D, float thr, int cw, int lane,
                                                int& flags, const float* srec, int c0, const Dir0Tab tab) {
  int cnt = 0;
  CellWalk cwk(cw + lane, S.gw);
  const bool wide = S.gw >= 32;
#pragma unroll 1
  for (int g = 0; g < kLiftPerThread; g += kCountGroup) {
    if (cw + g * 32 >= S.cells) break;  // uniform across the warp
    int idx[kCountGroup];
    bool kp[kCountGroup];
#pragma unroll
    for (int j = 0; j < kCountGroup; ++j, wide ? cwk.next_wide(S.gw) : cwk.next(S.gw)) {
      kp[j] = false;
      idx[j] = 0;
      if (cwk.cell < S.cells) {
        const float* r = srec + 3 * (cwk.cell - c0);
        const float c = r[2], tx = r[0], ty = r[1];
        flags |= content_flags_f(c, tx, ty);
        bool keep = gate<float>(c, thr);
        if (KIND != kGateOnly) {
          if (DIR == 0) {
            if (tab.on) {
              idx[j] = tab.iy[cwk.row - tab.row0] * D.w + tab.ix[cwk.col];
            } else {
              double sx, sy;
              source_px(S, cwk.row, cwk.col, sx, sy);
              idx[j] = direct_idx(D, sx, sy);
            }
          } else {
            const Bilin b = bilin(D, dmul((double)tx, D.sxd), dmul((double)ty, D.syd));
            keep = keep && b.inside;
            idx[j] = b.i00;
          }
        }
        kp[j] = keep;
        if (!keep) idx[j] = 0;
      }
    }
    if (KIND == kGateOnly) {
#pragma unroll
      for (int j = 0; j < kCountGroup; ++j) cnt += kp[j] ? 1 : 0;
    } else if (DIR == 0) {
      bool ok[kCountGroup];
#pragma unroll
      for (int j = 0; j < kCountGroup; ++j) ok[j] = tap_ok<KIND>(D, idx[j]);
#pragma unroll
      for (int j = 0; j < kCountGroup; ++j) cnt += (kp[j] && ok[j]) ? 1 : 0;
    } else {
      bool ok[kCountGroup][4];
#pragma unroll
      for (int j = 0; j < kCountGroup; ++j) {
        ok[j][0] = tap_ok<KIND>(D, idx[j]);
        ok[j][1] = tap_ok<KIND>(D, idx[j] + 1);
        ok[j][2] = tap_ok<KIND>(D, idx[j] + D.w);
        ok[j][3] = tap_ok<KIND>(D, idx[j] + D.w + 1);
      }
#pragma unroll
      for (int j = 0; j < kCountGroup; ++j) cnt += (kp[j] && ok[j][0] && ok[j][1] && ok[j][2] && ok[j][3]) ? 1 : 0;
    }
  }
  return cnt;
}

template <typename T>
__global__ void __launch_bounds__(kLiftThreads, VL_LIFT_CMINB) k_lift_count(LiftArgs a, int mode, int grouped) {
  const int64_t b = blockIdx.x;
  const int s = __ldg(a.seg_of_blk + b);  // host-built tile -> segment table (no per-thread binary search)
  const SegP S = load_seg(a.segs + s);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c0 = (int)(b - a.seg_blk0[s]) * kLiftBlockCells;
  const int cw = c0 + wid * kLiftWarpCells;
  const T thr = (T)a.threshold;
  __shared__ __align__(16) float srec_buf[3 * kLiftBlockCells];
  __shared__ __align__(8) uint64_t sbar;
  __shared__ int s_ix[kTabCols], s_iy[kTabRows];
  DepP D{};
  int kind = kGateOnly;
  Dir0Tab tab;
  tab.on = false;
  if (mode == 0) {
    const LiftDepth* gd = a.depths + S.depth;
    D = load_dep(gd);
    kind = __ldg(&gd->kind);
    fill_dir0_tab(S, D, c0, false, s_ix, s_iy, nullptr, nullptr, tab);
  }
  const float* srec = stage_records(S, c0, srec_buf, &sbar);  // its barrier also publishes the tables
  Dir0Tab notab = tab;
  notab.on = false;
  int cnt = 0, flags = 0;
  if (cw < S.cells && srec && grouped) {
    // staged IMLC records are f32 (T = float for them)
#define VL_LIFT_COUNT2(K)                                                                                   \
  cnt = S.direction == 0 ? count_run_staged<0, K>(S, D, (float)thr, cw, lane, flags, srec, c0, tab)         \
                         : count_run_staged<1, K>(S, D, (float)thr, cw, lane, flags, srec, c0, notab);
    switch (kind) {
      case kDepthF32: VL_LIFT_COUNT2(kDepthF32) break;
      case kDepthF16: VL_LIFT_COUNT2(kDepthF16) break;
      case kDepthCode8: VL_LIFT_COUNT2(kDepthCode8) break;
      case kDepthCode16: VL_LIFT_COUNT2(kDepthCode16) break;
      default: cnt = count_run_staged<0, kGateOnly>(S, D, (float)thr, cw, lane, flags, srec, c0, notab); break;
    }
#undef VL_LIFT_COUNT2
  } else if (cw < S.cells) {
#define VL_LIFT_COUNT(K)                                                                       \
  cnt = S.direction == 0 ? count_run<T, 0, K>(S, D, thr, cw, lane, flags, srec, c0, tab)         \
                         : count_run<T, 1, K>(S, D, thr, cw, lane, flags, srec, c0, notab);
    switch (kind) {
      case kDepthF32: VL_LIFT_COUNT(kDepthF32) break;
      case kDepthF16: VL_LIFT_COUNT(kDepthF16) break;
      case kDepthCode8: VL_LIFT_COUNT(kDepthCode8) break;
      case kDepthCode16: VL_LIFT_COUNT(kDepthCode16) break;
      default: cnt = count_run<T, 0, kGateOnly>(S, D, thr, cw, lane, flags, srec, c0, notab); break;
    }
#undef VL_LIFT_COUNT
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

// Exclusive scan of the block counts: one 1024-thread CTA per chunk of 1024
// blocks writes chunk-relative offsets and the chunk total; the last CTA to
// finish (atomic ticket) scans the chunk totals and writes the segment
// offsets, the total and the host mirrors.  (A single CTA walking 35840
// blocks took 43-85 us at C5.)
constexpr int kScanChunk = 1024;

__global__ void __launch_bounds__(kScanChunk) k_lift_scan(LiftArgs a) {
  __shared__ int64_t wtot[32];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * kScanChunk + threadIdx.x;
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
    const int64_t t = wtot[w];
    if (w < wid) wb += t;
    tot += t;
  }
  if (i < a.nblk) a.blk_off[i] = wb + x - v;
  if (threadIdx.x == 0) a.chunk_off[blockIdx.x] = tot;  // the chunk total for now
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.scan_ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // chunk totals -> exclusive chunk offsets: one block-wide scan per 1024 chunks
  int64_t carry = 0;
  for (unsigned k0 = 0; k0 < gridDim.x; k0 += kScanChunk) {
    const unsigned k = k0 + threadIdx.x;
    const int64_t cv = k < gridDim.x ? __ldcg(a.chunk_off + k) : 0;
    int64_t cx = cv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, cx, o);
      if (lane >= o) cx += y;
    }
    __syncthreads();
    if (lane == 31) wtot[wid] = cx;
    __syncthreads();
    int64_t cb = 0, ct = 0;
    for (int w = 0; w < 32; ++w) {
      const int64_t t = wtot[w];
      if (w < wid) cb += t;
      ct += t;
    }
    if (k < gridDim.x) a.chunk_off[k] = carry + cb + cx - cv;
    carry += ct;
  }
  if (threadIdx.x == 0) {
    a.seg_off[a.nseg] = carry;
    if (a.seg_off_host) a.seg_off_host[a.nseg] = carry;
  }
  __threadfence_block();
  __syncthreads();
  for (int s = threadIdx.x; s < a.nseg; s += kScanChunk) {
    const int64_t b0 = a.seg_blk0[s];
    const int64_t o = __ldcg(a.chunk_off + b0 / kScanChunk) + __ldcg(a.blk_off + b0);
    a.seg_off[s] = o;
    if (a.seg_off_host) a.seg_off_host[s] = o;
    if (a.seg_flags_host) a.seg_flags_host[s] = a.seg_flags ? __ldcg(a.seg_flags + s) : 0;
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

// Write pass: recompute the keep decision, lift the kept cells and store
// them at their ranked rows (a warp's rows are consecutive: every store
// instruction covers one contiguous run; staging the 24-B X rows through
// shared memory for unit-stride stores measured 2.6 % slower — the pass is
// issue-bound, not store-bound).
template <typename T, int DIR, int KIND>
__device__ __forceinline__ void write_run(const LiftArgs& a, const SegP& S, const DepP& D, const double* R,
                                          const double* t, T thr, int cw, int lane, int64_t pos,
                                          const float* srec, int c0, const Dir0Tab tab) {
  const unsigned lt = (1u << lane) - 1u;
  // the capacity clip only matters when the caller's arrays are too small
  const bool room = pos + kLiftWarpCells <= a.capacity;
  CellWalk cwk(cw + lane, S.gw);
  for (int i = 0; i < kLiftPerThread; ++i, cwk.next(S.gw)) {
    if (cw + i * 32 >= S.cells) break;  // uniform across the warp
    bool keep = false;
    double px0 = 0, px1 = 0, X0 = 0, X1 = 0, X2 = 0, wv = 0;
    if (cwk.cell < S.cells) {
      T c;
      double tx, ty;
      load_cell<T>(S, cwk.cell, c, tx, ty, srec, c0);
      keep = gate<T>(c, thr);
      wv = (double)c;
      if (keep) {
        if (KIND == kGateOnly) {
          source_px(S, cwk.row, cwk.col, px0, px1);
          X0 = tx;
          X1 = ty;
          X2 = (double)cwk.cell;
        } else if (DIR == 0) {
          // db -> query: direct lookup at the db cell (localizer.py:164-177)
          bool ok;
          double X[3];
          if (tab.on) {
            const int r = cwk.row - tab.row0;
            const double d = (double)tap_val<KIND>(D, tab.iy[r] * D.w + tab.ix[cwk.col], ok);
            if (ok) lift_point_n(R, t, tab.xn[cwk.col], tab.yn[r], d, X);
          } else {
            double sx, sy;
            source_px(S, cwk.row, cwk.col, sx, sy);
            const double d = (double)tap_val<KIND>(D, direct_idx(D, sx, sy), ok);
            if (ok) lift_point(D, R, t, sx, sy, d, X);
          }
          keep = ok;
          if (ok) {
            X0 = X[0];
            X1 = X[1];
            X2 = X[2];
            px0 = tx;
            px1 = ty;
          }
        } else {
          // query -> db: bilinear at the subpixel target (localizer.py:181-196)
          double d;
          keep = interp_val<KIND>(D, dmul(tx, D.sxd), dmul(ty, D.syd), d);
          if (keep) {
            double X[3];
            lift_point(D, R, t, tx, ty, d, X);
            X0 = X[0];
            X1 = X[1];
            X2 = X[2];
            source_px(S, cwk.row, cwk.col, px0, px1);
          }
        }
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    const int nk = __popc(m);
    if (keep) {
      const int k = __popc(m & lt);
      const int64_t p = pos + k;
      if (room || p < a.capacity) {
        a.X_out[3 * p] = X0;
        a.X_out[3 * p + 1] = X1;
        a.X_out[3 * p + 2] = X2;
        reinterpret_cast<double2*>(a.px_out)[p] = make_double2(px0, px1);
        a.w_out[p] = wv;
        if (a.entry_out) a.entry_out[p] = S.entry;
      }
    }
    pos += nk;
  }
}

template <typename T>
__global__ void __launch_bounds__(kLiftThreads, VL_LIFT_WMINB) k_lift_write(LiftArgs a, int mode) {
  __shared__ __align__(16) float srec_buf[3 * kLiftBlockCells];
  __shared__ __align__(8) uint64_t sbar;
  __shared__ double sRt[12];  // the database pose (block-uniform broadcast reads)
  __shared__ int s_ix[kTabCols], s_iy[kTabRows];
  __shared__ double s_xn[kTabCols], s_yn[kTabRows];
  const int64_t b = blockIdx.x;
  const int s = __ldg(a.seg_of_blk + b);  // host-built tile -> segment table (no per-thread binary search)
  const SegP S = load_seg(a.segs + s);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c0 = (int)(b - a.seg_blk0[s]) * kLiftBlockCells;
  const int cw = c0 + wid * kLiftWarpCells;
  const T thr = (T)a.threshold;
  DepP D{};
  int kind = kGateOnly;
  Dir0Tab tab;
  tab.on = false;
  if (mode == 0) {
    const LiftDepth* gd = a.depths + S.depth;
    D = load_dep(gd);
    kind = __ldg(&gd->kind);
    if (threadIdx.x < 12) sRt[threadIdx.x] = threadIdx.x < 9 ? __ldg(gd->R + threadIdx.x) : __ldg(gd->t + threadIdx.x - 9);
    fill_dir0_tab(S, D, c0, true, s_ix, s_iy, s_xn, s_yn, tab);
  }
  const float* srec = stage_records(S, c0, srec_buf, &sbar);  // its barrier also publishes sRt and the tables
  if (cw >= S.cells) return;  // whole warp past the segment end
  // this warp's first output row: block offset + the block's earlier warps
  int64_t pos = a.blk_off[b] + a.chunk_off[b / kScanChunk];
  {
    const int c = lane < wid ? a.warp_count[b * kLiftWarps + lane] : 0;
    pos += warp_sum(c);
  }
  Dir0Tab notab = tab;
  notab.on = false;
  const double* R = sRt;
  const double* t = sRt + 9;
#define VL_LIFT_WRITE(K)                                                                                 \
  if (S.direction == 0) write_run<T, 0, K>(a, S, D, R, t, thr, cw, lane, pos, srec, c0, tab);    \
  else write_run<T, 1, K>(a, S, D, R, t, thr, cw, lane, pos, srec, c0, notab);
  switch (kind) {
    case kDepthF32: VL_LIFT_WRITE(kDepthF32) break;
    case kDepthF16: VL_LIFT_WRITE(kDepthF16) break;
    case kDepthCode8: VL_LIFT_WRITE(kDepthCode8) break;
    case kDepthCode16: VL_LIFT_WRITE(kDepthCode16) break;
    default: write_run<T, 0, kGateOnly>(a, S, D, nullptr, nullptr, thr, cw, lane, pos, srec, c0, notab); break;
  }
#undef VL_LIFT_WRITE
}

int launch_lift(const LiftArgs& a, int field_f64, int mode, cudaStream_t st) {
  if (a.nblk <= 0) return 0;
  // VISLOC_LIFT_GROUPED=0: the per-cell count loop (A/B switch, read once)
  static const int grouped = [] {
    const char* e = getenv("VISLOC_LIFT_GROUPED");
    return e ? atoi(e) : 1;
  }();
  if (field_f64) k_lift_count<double><<<(unsigned)a.nblk, kLiftThreads, 0, st>>>(a, mode, grouped);
  else k_lift_count<float><<<(unsigned)a.nblk, kLiftThreads, 0, st>>>(a, mode, grouped);
  k_lift_scan<<<(unsigned)((a.nblk + kScanChunk - 1) / kScanChunk), kScanChunk, 0, st>>>(a);
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
