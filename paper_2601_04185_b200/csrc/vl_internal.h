// Internal declarations shared by the kernel translation units and the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "vl_common.cuh"
#include "vl_rng.cuh"

namespace vl {

constexpr int kMaxDevices = 64;  // per-device launch state (function attributes)

// Scoring tile geometry (vl_score.cu).
constexpr int kScoreThreads = 128;
#ifndef VL_SCORE_HT
#define VL_SCORE_HT 6
#endif
constexpr int kScoreHypPerThread = VL_SCORE_HT;  // coarse items: hypotheses per thread (sweeps: tools/)
constexpr int kScoreTileHyps = kScoreThreads * kScoreHypPerThread;  // 768
#ifndef VL_SCORE_SPI
#define VL_SCORE_SPI 4
#endif
constexpr int kScoreItemSplits = VL_SCORE_SPI;  // coarse items: 4 splits = 512 correspondences
// canonical cost = sum over split groups (in order) of the group sum
// ((p0 + p1) + p2) + p3 over its splits; coarse items produce one group
constexpr int kGroupSplits = kScoreItemSplits;
constexpr int kScoreHypPerThreadFine = 2;  // fine items (small batches): 1 pair, 1 split
constexpr int kScoreTileHypsFine = kScoreThreads * kScoreHypPerThreadFine;  // 256
// correspondences per split: the canonical fp32 summation unit (each split is
// summed sequentially by one thread, splits are combined in order by k_scan),
// so the cost bits do not depend on the tile shape, item size or grid
constexpr int kScoreChunk = 128;

// fp32 scoring rows: 0 = the scorer reads them at their solution slot
// through hsrc; 1 = k_compact copies them into hypothesis order first (A/B,
// ms per step C3 / C3 pruned: 93.3 / 48.5 vs 93.1 / 49.6: the copy costs
// 0.9 ms of compaction per step and saves ~1 ms of full scoring rounds only)
#ifndef VL_P32_COPY
#define VL_P32_COPY 0
#endif

// Per-query device state of the batched estimator.
struct __align__(16) QState {
  GenState gen;        // initial generator state
  // sampler cache: the PCG64 state advanced m_cache steps from gen.state (the
  // base of the last speculation window; m_cache = ~0: none), so the next
  // round's base is a short table jump instead of an O(log n) advance
  u128 st_cache;
  uint64_t m_cache;
  int64_t off;         // first row in px/X/w (absolute)
  int64_t coff;        // first row in the chunk-relative compaction buffer
  int64_t sub_off;     // first row in the scoring-subset arrays
  int n, nsub, stride, nsplit;
  Intr in;
  // dynamic
  uint64_t rng_pos;    // uint32 words consumed so far (the sampler's own chain)
  int64_t iters;       // minimal samples drawn in the rounds scanned so far (committed by k_scan)
  int64_t spec_iters;  // samples drawn by the sampler so far (may run one round ahead, see below)
  // per round parity (Work::par): samples of that round and the sample count
  // after it.  The pipelined loop (small batches) samples and solves round
  // r+1 on a side stream while round r is scored and scanned, so the
  // sampler's outputs are double-buffered and k_scan commits `iters`.
  int64_t iters_p[2];
  int bn_p[2];
  int active;
  int has_best;
  int nh;              // hypotheses in the current round
  double best_cost;
  Pose best;
  int64_t lo_calls, hyps, evals, rounds;
  // subset inlier count of `best` (the stop rule's msac_score, posest.py:269-273),
  // kept while `best` is unchanged: the next rounds' stop checks reuse it
  int64_t best_sub_cnt;
  int best_cnt_valid, pad_;
  // exact scoring pruning (vl_score.cuh): prune_ok = every fp32 subset weight
  // is >= 0 (MSAC partial sums then only grow), cost_typ = mean fp32 cost of
  // the last fully scored round, sA = splits scored for EVERY hypothesis this
  // round (the rest only for hypotheses whose prefix is below best_cost)
  float cost_typ;
  int sA, prune_ok;
  int nsurv, tiles_closed;  // this round's surviving hypotheses / closed scoring tiles (reset by k_compact)
  float prune_m;            // prefix margin (x best / typical cost), raised when many hypotheses survive
  int h_lo, h_hi;           // hypotheses [h_lo, h_hi) scored / scanned in this launch phase (head / rest / full)
};

struct ScoreItem {
  int q, tile, split, nsplit;  // query, hypothesis tile, first split, splits in the item
};

// Scoring tail task (pruned rounds): up to 32 surviving hypotheses of one
// query, listed at surv[q][base .. base + cnt), finished over splits [sA, NS).
struct TailTask {
  int q, base, cnt, pad;
};

struct RansacParams {
  int64_t max_iterations;
  int batch_size;
  int lm_max_iters;
  double eta;
  double tau;
  double cauchy;
};

// Device workspace view for one chunk of queries.
constexpr int kGeoDoubles = 25;  // sizeof(P3PGeo) / 8
constexpr int kMaxCandSlots = 8;  // distance-triple candidates per sample (4 roots x 2 branches)

struct Work {
  QState* qs;
  int* active_list;
  int* active_count;     // device scalar
  int* next_active;      // [Qc]
  int* samples;          // [Qc][B][3]
  double* slots;         // [Qc][ceil(B/32)][4 * 12][32] solution slots (R row-major + t), warp-blocked SoA
  int* slot_cnt;         // [Qc][B]
  // P3P scratch (k_p3p_roots -> k_p3p_polish), warp-blocked SoA: samples are
  // grouped 32 per block (group = q * ceil(B/32) + s/32, lane = s % 32) and
  // field f of a sample lives at [group][f][lane], so a warp's stores and
  // loads of one field are 256 contiguous bytes
  double* p3p_geo;       // [Qc][ceil(B/32)][kGeoDoubles][32] per-sample geometry
  double* p3p_cand;      // [Qc][ceil(B/32)][8 * 3][32] distance-triple candidates
  int* p3p_nc;           // [Qc][B] candidate counts
  float* P32;            // [Qc][12][HCAP] fp32 scoring rows in hypothesis order (k_compact)
  float* P32s;           // [Qc][12][4][B]  the same rows at their solution slot, column k * B + s (k_p3p_polish)
  int* hsrc;             // [Qc][HCAP]
  ScoreItem* items;      // [item_cap]
  int* item_count;       // [0] items appended this round, [1] scoring work cursor, [2] k_scan completion ticket,
                         // [3] scoring tail tasks
  float* partial;        // [Qc][NSPLIT][HCAP] split / group partial sums
  float* cost32;         // [Qc][HCAP] final fp32 costs (written by the last item of each tile)
  int* tile_cnt;         // [Qc][TCAP] per-round completion tickets of the scoring tiles
  double2* sub_pk;       // [Nsub][3] packed fp64 scoring subset: (X,Y) (Z,u) (v,w)
  float4* sub32;         // [Nsub/2][3] record pairs (SoA float2), per-query offsets even
  double2* comp_pk;      // [N][3] packed full-set inliers (final refinement)
  int B, HCAP, NSPLIT, TCAP;
  int64_t item_cap;
  int split_rank, split_size;  // hypothesis-split mode: scoring tiles dealt round-robin
  int par;               // round parity: selects bn_p / iters_p (0 unless pipelined)
  int* next_list;        // k_scan's compaction target (== active_list: in place)
  int* next_count;       // (== active_count)
  int* host_count;       // mapped pinned mirror of *active_count (nullable)
  u128* jump;            // [Qc][2][kJumpBits] per-query PCG64 jump tables (k_prep; nullable)
  // exact scoring pruning (coarse rounds with a best pose; 0 = every
  // hypothesis scored on the whole subset, as the reference does)
  int prune;
  int* surv;                     // [Qc][HCAP] surviving hypotheses of each query (any order)
  TailTask* tail;                // [tail_cap] tasks (count: item_count[3])
  int64_t tail_cap;
  unsigned long long* prune_ctr; // [2] evaluations skipped / evaluated by the tail (run totals)
};

// Programmatic dependent launch (PDL): every kernel of the round loop waits
// for its predecessor grid's completion + memory flush at entry (a no-op when
// launched without the PDL attribute) and immediately lets its own dependent
// launch: for latency-bound small batches the next kernel's launch and CTA
// scheduling then overlap this kernel instead of following it.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Element e (0..11: R row-major, t) of solution k of sample s of query q in
// the warp-blocked slot layout: slot_ptr(...)[32 * e].
__device__ __forceinline__ double* slot_ptr(const Work& wk, int q, int s, int k) {
  return wk.slots + (((int64_t)q * ((wk.B + 31) / 32) + s / 32) * 48 + 12 * k) * 32 + (s & 31);
}

struct Inputs {
  const double* px;
  const double* X;
  const double* w;
};

struct Outputs {
  double* q;
  double* t;
  uint8_t* flags;
  int64_t* inlier_count;
  double* score;
  int64_t* iterations;
  int32_t* converged;
  int64_t* stats;
};

// ---- launchers (return number of kernels launched) -------------------------
int launch_prep(const Work& wk, const Inputs& in, int q0, int nq, int list_pos, const QState* host_qs,
                cudaStream_t st);
// profiling stages (vl_profile_read order)
enum { kStagePrep = 0, kStageSample, kStageP3P, kStageCompact, kStageScore, kStageScan, kStageActive,
       kStageFinal, kStageLift, kNumStages };
// VISLOC_CARVEOUT A/B knob (vl_ransac.cu)
int carveout_mode();
// fine scoring items (256-hypothesis tiles x 1 split) for a round of nactive queries
bool round_is_fine(const Work& wk, int nactive, int num_sms);
// phase 0: whole round; 1: sample .. score; 2: scan + active (stepwise driver);
// pipelined loop: 3 sampling + P3P, 4 compaction, 5 scores + scan.
// split (phase 0, pruning on, coarse rounds): queries without a best pose
// first score and scan their first kHeadHyps hypotheses, so the rest of the
// round is already pruned against that best (vl_ransac.cu, k_compact)
int launch_round(const Work& wk, const Inputs& in, const RansacParams& p, int nactive, int num_sms,
                 cudaStream_t st, void (*hook)(void*, int, bool), void* hook_arg, int phase, int split = 0);
int launch_final(const Work& wk, const Inputs& in, const Outputs& out, const RansacParams& p, int Q,
                 int q_base, cudaStream_t st);

int launch_msac(const Pose& pose, const double* px, const double* X, const double* w, int n, Intr in,
                double tau, double* red_out, uint8_t* flags, cudaStream_t st);
int launch_robust_cost(const Pose& pose, const double* px, const double* X, const double* w, int n, Intr in,
                       int kind, double scale, double* out, cudaStream_t st);
int launch_residuals(const Pose& pose, const double* px, const double* X, int n, Intr in, double* res, double* z,
                     double* J, cudaStream_t st);
int launch_refine(const Pose& start, const double* px, const double* X, const double* w, int n, Intr in,
                  int kind, double scale, int max_iters, double gtol, double ctol, Pose* pose_out,
                  int* info_out, double* trace, cudaStream_t st);
int launch_p3p_batch(const double* f, const double* P, int B, double* slots, int* cnt, double* R_out,
                     double* t_out, int64_t* idx_out, int* m_out, cudaStream_t st);
int launch_sample(const GenState& g, uint64_t pos0, int64_t n, int count, int* out, uint64_t* pos_out,
                  cudaStream_t st);

// standalone scoring: fp32 rows + score items of H caller hypotheses (query 0)
int launch_hyp_rows(const Work& wk, const double* R, const double* t, int H, int fine, cudaStream_t st);
int launch_score(const Work& wk, float tau2, int num_sms, int fine, int nactive, cudaStream_t st,
                 bool pdl = false);

// hypothesis-split packed (score, index) variant (vl_ransac.cu)
int launch_split_argmin(const Work& wk, int nactive, int num_sms, long long* keys, cudaStream_t st);
int launch_split_apply_argmin(const Work& wk, int nactive, const long long* keys, cudaStream_t st);
int launch_fill_i64(long long* p, int n, long long v, cudaStream_t st);

}  // namespace vl
