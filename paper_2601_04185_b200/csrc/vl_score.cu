// fp32 MSAC hypothesis scoring — the FP32 CUDA-core roofline kernel.
//
// Replaces posest._score_hypotheses (posest.py:178-220): for every hypothesis
// h and scoring correspondence i,
//     cost_h = sum_i w_i * min(e_i^2, tau^2),   behind-camera -> tau^2,
// in fp32 (ranking only; definitive costs come from the fp64 msac pass).
//
// Work decomposition: a work item is (query, tile of 768 hypotheses, split of
// 512 correspondences).  A persistent grid (SMs x resident CTAs) walks the
// item list; each thread keeps 6 hypotheses' fx/fy-folded [R|t] rows as three
// f32x2 pairs in registers and streams the split's correspondence records
// from shared memory (broadcast reads: all lanes read the same record).
// Per pair of evaluations (FFMA2 / FMUL2 = Blackwell packed FP32):
//     x,y,z  = 9 FFMA2 (P row . [X Y Z] + P03, coordinate broadcast operand)
//     r      = MUFU.RSQ x2, FMUL2 (r = rsqrt(z)^2: NaN for z<0, inf for z==0)
//     du,dv  = 2 FFMA2 (x*r + (cx-u)), (y*r + (cy-v))
//     e2     = FMUL2 + FFMA2
//     min    = FMNMX x2 (minNum: NaN/inf -> tau^2 handles behind-camera)
//     acc   += FFMA2(w, min)
// = 15 FMA-pipe instructions per 2 evaluations (30 FLOP/eval).
// Split partial sums land in partial[q][split][h] and are reduced in fixed
// split order by k_scan, so costs do not depend on the launch geometry.
// Variant sweep and ncu evidence: tools/score_bench.cu, profiles/.
#include "vl_score.cuh"

namespace vl {

constexpr int kScoreMinBlocks = 3;
constexpr int kScoreUnroll = 2;

int launch_score(const Work& wk, float tau2, int num_sms, cudaStream_t st) {
  auto kern = k_score2_t<kScoreThreads, kScoreHypPerThread, kScoreChunk, kScoreMinBlocks, kScoreUnroll>;
  static int occ = 0;
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kScoreThreads, 0) != cudaSuccess || occ < 1)
      occ = kScoreMinBlocks;
  }
  kern<<<num_sms * occ, kScoreThreads, 0, st>>>(wk, tau2);
  return 1;
}

}  // namespace vl
