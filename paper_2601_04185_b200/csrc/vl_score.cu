// fp32 MSAC hypothesis scoring — the FP32 CUDA-core roofline kernel.
//
// Replaces posest._score_hypotheses (posest.py:178-220): for every hypothesis
// h and scoring correspondence i,
//     cost_h = sum_i w_i * min(e_i^2, tau^2),   behind-camera -> tau^2,
// in fp32 (ranking only; definitive costs come from the fp64 msac pass).
//
// Work decomposition: a work item is (query, tile of 512 hypotheses, split of
// 512 correspondences).  A persistent grid walks the item list; each thread
// keeps 4 hypotheses' fx/fy-folded [R|t] rows (48 floats) in registers and
// streams the split's correspondence records from shared memory (broadcast
// reads: all lanes read the same record).  Per evaluation:
//     x,y,z  = 9 FFMA (P row . [X Y Z] + P03)
//     r      = rsqrt(z)^2 (MUFU.RSQ + FMUL; NaN for z<0, inf for z==0)
//     du,dv  = 2 FFMA (x*r + (cx-u)), (y*r + (cy-v))
//     e2     = FMUL + FFMA
//     min    = FMNMX (minNum: NaN -> tau^2 handles behind-camera)
//     acc   += FFMA(w, min)
// = 15 FMA-pipe + 1 MUFU + 1 ALU instructions per evaluation.
// Split partial sums land in partial[q][split][h] and are reduced in fixed
// split order by k_scan, so costs do not depend on the launch geometry.
#include "vl_internal.h"

namespace vl {

__device__ __forceinline__ float rsqrt_approx_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int HT>
__global__ void __launch_bounds__(kScoreThreads, 4) k_score(Work wk, float tau2) {
  __shared__ float4 rec[2 * kScoreChunk];
  const int nitems = *wk.item_count;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const ScoreItem item = wk.items[it];
    const QState& S = wk.qs[item.q];
    const int nh = S.nh, nsub = S.nsub;
    const int c0 = item.split * kScoreChunk;
    const int cn = min(kScoreChunk, nsub - c0);
    const float4* src = wk.sub32 + 2 * (S.sub_off + c0);
    __syncthreads();
    for (int k = threadIdx.x; k < 2 * cn; k += kScoreThreads) rec[k] = src[k];
    float P[HT][12];
    int hid[HT];
    const float* Pq = wk.P32 + (int64_t)item.q * 12 * wk.HCAP;
#pragma unroll
    for (int j = 0; j < HT; ++j) {
      const int h = item.tile * kScoreTileHyps + j * kScoreThreads + threadIdx.x;
      hid[j] = h;
      const int hc = h < nh ? h : 0;
#pragma unroll
      for (int c = 0; c < 12; ++c) P[j][c] = Pq[(int64_t)c * wk.HCAP + hc];
    }
    __syncthreads();
    float acc[HT];
#pragma unroll
    for (int j = 0; j < HT; ++j) acc[j] = 0.f;
#pragma unroll 2
    for (int c = 0; c < cn; ++c) {
      const float4 a = rec[2 * c];
      const float4 b = rec[2 * c + 1];
#pragma unroll
      for (int j = 0; j < HT; ++j) {
        const float x = fmaf(P[j][0], a.x, fmaf(P[j][1], a.y, fmaf(P[j][2], a.z, P[j][3])));
        const float y = fmaf(P[j][4], a.x, fmaf(P[j][5], a.y, fmaf(P[j][6], a.z, P[j][7])));
        const float z = fmaf(P[j][8], a.x, fmaf(P[j][9], a.y, fmaf(P[j][10], a.z, P[j][11])));
        const float rs = rsqrt_approx_ftz(z);
        const float r = rs * rs;
        const float du = fmaf(x, r, a.w);
        const float dv = fmaf(y, r, b.x);
        const float e2 = fminf(fmaf(du, du, dv * dv), tau2);
        acc[j] = fmaf(b.y, e2, acc[j]);
      }
    }
    float* out = wk.partial + ((int64_t)item.q * wk.NSPLIT + item.split) * wk.HCAP;
#pragma unroll
    for (int j = 0; j < HT; ++j)
      if (hid[j] < nh) out[hid[j]] = acc[j];
  }
}

int launch_score(const Work& wk, float tau2, int num_sms, cudaStream_t st) {
  // persistent: 4 resident CTAs per SM
  const int grid = num_sms * 4;
  k_score<kScoreHypPerThread><<<grid, kScoreThreads, 0, st>>>(wk, tau2);
  return 1;
}

}  // namespace vl
