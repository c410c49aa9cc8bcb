// Internal structures of the depth-lifting kernels (vl_lift.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vl {

enum { kDepthF32 = 0, kDepthF16 = 1, kDepthCode8 = 2, kDepthCode16 = 3 };

// One database entry's stored depth + camera (device copy of vl_lift_depth).
struct LiftDepth {
  int w, h, kind, pad;
  const void* values;    // f32 / f16 values, or u8 / u16 codes
  const uint8_t* valid;  // kinds f32 / f16
  const float* lut;      // kinds code8 / code16: code -> f32 depth (code 0 invalid)
  double fx, fy, cx, cy;
  double sx_depth, sy_depth;
  double R[9], t[3];
};

// One correspondence field in output order (device copy of vl_lift_segment).
enum { kLayoutPlanar = 0, kLayoutImlc = 1 };
enum { kFieldBadConf = 1, kFieldBadTarget = 2 };

struct LiftSeg {
  int query, entry, direction, depth;
  int gw, gh;
  int layout, pad;
  double scale_x, scale_y;
  const void* targets;     // planar: [gh*gw*2] f32 or f64; IMLC: [gh*gw*3] f32 records
  const void* confidence;  // planar: [gh*gw]
};

struct LiftArgs {
  const LiftSeg* segs;
  int nseg;
  const LiftDepth* depths;
  const int64_t* seg_blk0;  // [nseg] first block of each segment
  int64_t nblk;
  int* blk_count;           // [nblk]
  int* warp_count;          // [nblk * 8] kept cells of every warp's 256-cell run
  int* seg_flags;           // [nseg] IMLC content verdicts (VL_FIELD_*), zeroed by the caller
  int64_t* blk_off;         // [nblk]
  int64_t* seg_off;         // [nseg+1]
  int64_t* seg_off_host;    // [nseg+1] mapped pinned mirror (nullable)
  int* seg_flags_host;      // [nseg]   mapped pinned mirror (nullable)
  double threshold;
  double* px_out;
  double* X_out;
  double* w_out;
  int32_t* entry_out;
  int64_t capacity;
  const int* seg_of_blk;    // [nblk] segment of every 2048-cell block (host-built)
  int64_t* chunk_off;       // [nchunk] offsets of the scan's 1024-block chunks (blk_off is chunk-relative)
  int* scan_ticket;         // zeroed by the caller
};

// copies `bytes` (multiple of 8) from mapped pinned host memory and zeroes
// zero_n ints — no copy-engine transfer on the stream
int launch_lift_prep(void* dst, const void* src_host, size_t bytes, int* zero, int zero_n, cudaStream_t st);
int launch_lift(const LiftArgs& a, int field_f64, int mode, cudaStream_t st);
int launch_lift_write(const LiftArgs& a, int field_f64, int mode, cudaStream_t st);
int lift_block_cells();
int launch_interp(const LiftDepth& D, const double* pts, int n, double* vals, uint8_t* ok, cudaStream_t st);
int launch_decode(const LiftDepth& D, int64_t n, float* vals, uint8_t* valid, cudaStream_t st);

}  // namespace vl
