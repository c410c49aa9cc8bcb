// Depth-map codecs: log quantisation of f32/f16 depth and the compression
// sweep's block reduction of codes.
//
// Reference: mapstore.quantize_depth (mapstore.py:96-119),
// _downsample_codes_nearest_valid (:390-414), _requantize_codes (:417-425).
//
// quantize: the reference maps an f32 depth through fp64 log / floor.  The
// code is a monotone step function of the f32 value, so the host tabulates its
// levels-1 step positions once with the reference's own arithmetic (the
// smallest f32 reaching each code, `mapstore.quantize_thresholds`) and the
// kernel counts thresholds <= value by binary search: bit-exact for every f32
// input, no transcendental on the device.  HBM-bound: 4 (or 2) + 1 B read,
// 1 (or 2) B written per pixel; the table sits in shared memory up to 12k
// levels, else in L1/L2.
//
// reduce: one thread per output cell scans its factor x factor block in
// row-major order keeping the valid code with the smallest squared distance
// to the block centre (strict <, so the first row-major minimum wins — the
// reference's argmin); distances are taken in doubled integer coordinates
// (exactly 4x the reference's fp64 values).  Requantisation uses the
// reference's fp64 operation order with explicit round-to-nearest intrinsics
// (no FMA contraction).
#include <algorithm>
#include <climits>
#include <cuda_fp16.h>
#include "vl_common.cuh"

namespace vl {

constexpr int kCodecThreads = 256;
constexpr int kCodecMaxJobs = 64;
constexpr int kCodecSmemThr = 12288;  // thresholds held in shared memory (48 KB)

struct CodecJob {
  int32_t w, h, kind, levels;
  const void* values;
  const uint8_t* valid;
  void* out;
};
struct CodecBatch {
  CodecJob j[kCodecMaxJobs];
};

__device__ __forceinline__ uint32_t count_le(const uint32_t* thr, int n, uint32_t bits) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (thr[mid] <= bits) lo = mid + 1;
    else hi = mid;
  }
  return (uint32_t)lo;
}

__global__ void __launch_bounds__(kCodecThreads) k_quantize(const __grid_constant__ CodecBatch b,
                                                            const uint32_t* __restrict__ thr, int nthr,
                                                            int out16) {
  extern __shared__ uint32_t s_thr[];
  const bool in_smem = nthr <= kCodecSmemThr;
  if (in_smem) {
    for (int i = threadIdx.x; i < nthr; i += blockDim.x) s_thr[i] = thr[i];
    __syncthreads();
  }
  const uint32_t* T = in_smem ? s_thr : thr;
  const CodecJob& J = b.j[blockIdx.y];
  const int64_t n = (int64_t)J.w * J.h;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t code = 0;
    if (J.valid[i]) {
      // valid pixels hold positive finite depth (DepthMap invariant): the
      // IEEE bit pattern orders like the value
      const float v = J.kind == 0 ? ((const float*)J.values)[i] : __half2float(((const __half*)J.values)[i]);
      code = 1u + count_le(T, nthr, __float_as_uint(v));
    }
    if (out16) ((uint16_t*)J.out)[i] = (uint16_t)code;
    else ((uint8_t*)J.out)[i] = (uint8_t)code;
  }
}

__global__ void __launch_bounds__(kCodecThreads) k_reduce_codes(const __grid_constant__ CodecBatch b, int factor,
                                                                int new_levels) {
  const CodecJob& J = b.j[blockIdx.y];
  const int ow = (J.w + factor - 1) / factor, oh = (J.h + factor - 1) / factor;
  const int64_t n = (int64_t)ow * oh;
  const bool in16 = J.kind == 3, out16 = new_levels > 255;
  const bool requant = new_levels != J.levels;
  const double old_denom = (double)max(J.levels - 1, 1), scale = (double)(new_levels - 1);
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    const int br = (int)(o / ow), bc = (int)(o - (int64_t)br * ow);
    const int r0 = br * factor, r1 = min(r0 + factor, J.h);
    const int c0 = bc * factor, c1 = min(c0 + factor, J.w);
    const int cr = r1 - r0 - 1, cc = c1 - c0 - 1;  // doubled block centre
    int best = INT_MAX;
    uint32_t code = 0;
    for (int r = r0; r < r1; ++r) {
      const int64_t row = (int64_t)r * J.w;
      const int dr = 2 * (r - r0) - cr;
      for (int c = c0; c < c1; ++c) {
        const uint32_t v = in16 ? ((const uint16_t*)J.values)[row + c] : ((const uint8_t*)J.values)[row + c];
        if (v == 0) continue;
        const int dc = 2 * (c - c0) - cc;
        const int d2 = dr * dr + dc * dc;
        if (d2 < best) {
          best = d2;
          code = v;
        }
      }
    }
    if (requant && code) {
      const double u = __ddiv_rn((double)code - 1.0, old_denom);
      code = 1u + (uint32_t)floor(__dadd_rn(__dmul_rn(u, scale), 0.5));
    }
    if (out16) ((uint16_t*)J.out)[o] = (uint16_t)code;
    else ((uint8_t*)J.out)[o] = (uint8_t)code;
  }
}

static int codec_grid(int64_t cells, int num_sms) {
  const int64_t want = (cells + kCodecThreads - 1) / kCodecThreads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms * 8));
}

int launch_quantize(const CodecJob* jobs, int njobs, const uint32_t* thr, int nthr, int out16, int num_sms,
                    cudaStream_t st) {
  int launches = 0;
  for (int j0 = 0; j0 < njobs; j0 += kCodecMaxJobs) {
    CodecBatch b;
    const int nj = std::min(kCodecMaxJobs, njobs - j0);
    int64_t cells = 0;
    for (int k = 0; k < nj; ++k) {
      b.j[k] = jobs[j0 + k];
      cells = std::max(cells, (int64_t)b.j[k].w * b.j[k].h);
    }
    const size_t smem = nthr <= kCodecSmemThr ? (size_t)nthr * 4 : 0;
    dim3 grid(codec_grid(cells, (num_sms + nj - 1) / nj), nj);
    k_quantize<<<grid, kCodecThreads, smem, st>>>(b, thr, nthr, out16);
    ++launches;
  }
  return launches;
}

int launch_reduce_codes(const CodecJob* jobs, int njobs, int factor, int new_levels, int num_sms, cudaStream_t st) {
  int launches = 0;
  for (int j0 = 0; j0 < njobs; j0 += kCodecMaxJobs) {
    CodecBatch b;
    const int nj = std::min(kCodecMaxJobs, njobs - j0);
    int64_t cells = 0;
    for (int k = 0; k < nj; ++k) {
      b.j[k] = jobs[j0 + k];
      const int64_t ow = (b.j[k].w + factor - 1) / factor, oh = (b.j[k].h + factor - 1) / factor;
      cells = std::max(cells, ow * oh);
    }
    dim3 grid(codec_grid(cells, (num_sms + nj - 1) / nj), nj);
    k_reduce_codes<<<grid, kCodecThreads, 0, st>>>(b, factor, new_levels);
    ++launches;
  }
  return launches;
}

}  // namespace vl
