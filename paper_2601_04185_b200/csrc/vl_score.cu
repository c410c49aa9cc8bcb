// fp32 MSAC hypothesis scoring — the FP32 CUDA-core roofline kernel.
//
// Replaces posest._score_hypotheses (posest.py:178-220): for every hypothesis
// h and scoring correspondence i,
//     cost_h = sum_i w_i * min(e_i^2, tau^2),   behind-camera -> tau^2,
// in fp32 (ranking only; definitive costs come from the fp64 msac pass).
//
// Work decomposition (vl_score.cuh): a work item is (query, tile of
// hypotheses, up to 4 splits of 128 correspondences).  A persistent grid
// (SMs x resident CTAs) walks the item list through a dynamic cursor; each
// thread keeps its hypotheses' fx/fy-folded [R|t] rows as f32x2 pairs in
// registers and streams the item's correspondence records from shared memory
// (broadcast reads: all lanes read the same record).  Per pair of
// evaluations (FFMA2 / FMUL2 = Blackwell packed FP32):
//     x,y,z  = 9 FFMA2 (P row . [X Y Z] + P03, coordinate broadcast operand)
//     r      = MUFU.RCP x2 of max(z, 0) (ALU clamp: +inf behind the camera)
//     du,dv  = 2 FFMA2 (x*r + (cx-u)), (y*r + (cy-v))
//     e2     = FMUL2 + FFMA2
//     min    = FMNMX x2 (minNum: NaN/inf -> tau^2 handles behind-camera)
//     acc   += FFMA2(w, min)
// = 14 FMA-pipe instructions per 2 evaluations (30 FLOP/eval).
// Each 128-record split is summed sequentially by one thread and lands in
// its own partial slot; k_scan adds the splits in order, so costs do not
// depend on the tile shape, the item size or the launch geometry.
// Variant sweep and ncu evidence: tools/score_bench.cu, profiles/.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include "vl_score.cuh"

namespace vl {

// coarse: 768-hypothesis tiles x 512 correspondences (big batches)
#ifndef VL_SCORE_UNR
#define VL_SCORE_UNR 2
#endif
constexpr int kCoarseMinBlocks = VL_SCORE_MINB;
// fine: 256-hypothesis tiles x 128 correspondences (single queries / small batches)
constexpr int kFineMinBlocks = 6;

// grid: persistent (SMs x resident CTAs, dynamic cursor) by default; the
// VISLOC_SCORE_GRID=items knob launches an item-count upper bound of CTAs
// instead (one item each) so that other streams' kernels can interleave.
// The persistent grid is capped at the round's item-count upper bound: a
// small round (C1: one query, 16 splits -> <= 256 fine items) launches no
// CTAs that would only find the cursor exhausted (C1 1.06 -> 0.94 ms).
static int score_grid(const Work& wk, int persistent, int fine, int nactive) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("VISLOC_SCORE_GRID");
    mode = (e && e[0] == 'i') ? 1 : 0;
  }
  const int tile = fine ? kScoreTileHypsFine : kScoreTileHyps, spi = fine == 1 ? 1 : kScoreItemSplits;
  const int64_t ub = (int64_t)nactive * ((wk.HCAP + tile - 1) / tile) * ((wk.NSPLIT + spi - 1) / spi);
  if (!mode) return (int)std::max<int64_t>(1, std::min<int64_t>(persistent, ub));
  return (int)std::min<int64_t>(ub, 1 << 30);
}

int launch_score(const Work& wk, float tau2, int num_sms, int fine, int nactive, cudaStream_t st, bool pdl) {
  // dynamic smem: the attribute is set once per device (host threads driving
  // separate contexts may get here together)
  static std::mutex mu;
  static bool attr_dev[kMaxDevices] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  constexpr size_t kFineSmem = score_smem_bytes<kScoreThreads, kScoreHypPerThreadFine, 1, kScoreChunk>();
  constexpr size_t kCoarseSmem = score_smem_bytes<kScoreThreads, kScoreHypPerThread, kScoreItemSplits, kScoreChunk>();
  auto fkern = k_score2_t<kScoreThreads, kScoreHypPerThreadFine, 1, kScoreChunk, kFineMinBlocks, 2, false>;
  auto mkern = k_score2_t<kScoreThreads, kScoreHypPerThreadFine, kScoreItemSplits, kScoreChunk, kFineMinBlocks, 2,
                          false>;
  constexpr size_t kMediumSmem = score_smem_bytes<kScoreThreads, kScoreHypPerThreadFine, kScoreItemSplits,
                                                  kScoreChunk>();
  auto ckern_full = k_score2_t<kScoreThreads, kScoreHypPerThread, kScoreItemSplits, kScoreChunk, kCoarseMinBlocks,
                               VL_SCORE_UNR, false>;
  auto ckern_prune = k_score2_t<kScoreThreads, kScoreHypPerThread, kScoreItemSplits, kScoreChunk, kCoarseMinBlocks,
                                VL_SCORE_UNR, true>;
  auto ckern = wk.prune ? ckern_prune : ckern_full;
  {
    std::lock_guard<std::mutex> g(mu);
    bool& a = attr_dev[dev < kMaxDevices ? dev : 0];
    if (!a) {
      cudaFuncSetAttribute(fkern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFineSmem);
      cudaFuncSetAttribute(mkern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMediumSmem);
      cudaFuncSetAttribute(ckern_full, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCoarseSmem);
      cudaFuncSetAttribute(ckern_prune, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCoarseSmem);
      if (carveout_mode()) {  // (see set_round_carveouts, vl_ransac.cu)
        const int v = cudaSharedmemCarveoutMaxShared;
        cudaFuncSetAttribute(fkern, cudaFuncAttributePreferredSharedMemoryCarveout, v);
        cudaFuncSetAttribute(ckern_full, cudaFuncAttributePreferredSharedMemoryCarveout, v);
        cudaFuncSetAttribute(ckern_prune, cudaFuncAttributePreferredSharedMemoryCarveout, v);
        cudaFuncSetAttribute(k_score_tail<kScoreThreads>, cudaFuncAttributePreferredSharedMemoryCarveout, v);
      }
      a = true;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kScoreThreads, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see pdl_enter (vl_internal.h)
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  if (fine == 2) {
    // medium items of a single query: one CTA per item (item upper bound)
    cfg.gridDim = dim3(score_grid(wk, num_sms * kFineMinBlocks, 2, nactive), 1, 1);
    cfg.dynamicSmemBytes = kMediumSmem;
    cudaLaunchKernelEx(&cfg, mkern, wk, tau2);
  } else if (fine) {
    static int occ = 0;
    if (occ == 0 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fkern, kScoreThreads, kFineSmem) !=
                         cudaSuccess || occ < 1))
      occ = kFineMinBlocks;
    // CTAs per SM of the fine grid: a single query's round (a few hundred
    // items) runs faster on 2 CTAs per SM than on all 6 (C4 5.82 -> 5.57 ms,
    // C2 1.22 -> 1.21; A/B knob VISLOC_SCORE_FINE_CTAS, 0 = occupancy)
    static int fine_ctas = -3;  // -3: not read yet; -2: automatic
    if (fine_ctas == -3) {
      const char* e = getenv("VISLOC_SCORE_FINE_CTAS");
      fine_ctas = e ? atoi(e) : -2;
    }
    const int want = fine_ctas == -2 ? (nactive == 1 ? 2 : 0) : fine_ctas;
    const int per_sm = want > 0 ? std::min(want, occ) : occ;
    cfg.gridDim = dim3(score_grid(wk, num_sms * per_sm, 1, nactive), 1, 1);
    cfg.dynamicSmemBytes = kFineSmem;
    cudaLaunchKernelEx(&cfg, fkern, wk, tau2);
  } else {
    static int occ = 0;
    if (occ == 0 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ckern, kScoreThreads, kCoarseSmem) !=
                         cudaSuccess || occ < 1))
      occ = kCoarseMinBlocks;
    cfg.gridDim = dim3(score_grid(wk, num_sms * occ, 0, nactive), 1, 1);
    cfg.dynamicSmemBytes = kCoarseSmem;
    cudaLaunchKernelEx(&cfg, ckern, wk, tau2);
    if (wk.prune) {
      // the survivors of pruned tiles (a few per query; no tasks in rounds
      // without a best pose): 8 CTAs of 4 warps per SM, one task per CTA at a time
      cfg.gridDim = dim3(8 * num_sms, 1, 1);
      cfg.dynamicSmemBytes = 0;
      cudaLaunchKernelEx(&cfg, k_score_tail<kScoreThreads>, wk, tau2);
      return 2;
    }
  }
  return 1;
}

}  // namespace vl
