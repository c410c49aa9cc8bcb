// C ABI (include/visloc_b200.h): context, workspace, and the host-side round
// loop of the batched estimator.  No CPU compute fallback exists: every
// entry point either launches sm_100a kernels or fails with a status code.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/visloc_b200.h"
#include "vl_internal.h"

using namespace vl;

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct vl_ctx {
  int device = 0;
  int num_sms = 148;
  std::string err;
  int64_t launches = 0;
  DevBuf qs, active, next_active, active_count, samples, slots, slot_cnt, p3p_geo, p3p_cand, p3p_nc, P32, P32s, hsrc, items, item_count,
      partial, cost32, tile_cnt, sub_pk, sub32, comp_pk;
  DevBuf surv, tail, prune_ctr;  // exact scoring pruning (vl_score.cuh)
  DevBuf jump;                   // per-query PCG64 jump tables
  // pipelined round loop (small batches): the parity-1 copies of the round
  // buffers, the second active list, the side stream and its events
  DevBuf samples2, slots2, slot_cnt2, p3p_geo2, p3p_cand2, p3p_nc2, P32s2, active2, active_count2;
  cudaStream_t side = nullptr;
  cudaEvent_t pev[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int prune = -1;                // -1: VISLOC_PRUNE (default on), else vl_set_scoring_pruning
  DevBuf scratch;  // small standalone-call scratch
  DevBuf lift_meta, lift_blk_count, lift_blk_off, lift_seg_off;  // vl_lift
  DevBuf tri_meta;                                               // vl_build_depth_maps
  void* h_pinned = nullptr;
  size_t h_pinned_cap = 0;
  // profiling: CUDA-event brackets around every stage launch (vl_profile)
  int prof = 0;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> ev_stage;  // stage of each recorded pair
  size_t ev_used = 0;
  double stage_ms[kNumStages] = {0};
  int64_t stage_launches[kNumStages] = {0};
  cudaStream_t prof_stream = nullptr;
  cudaEvent_t round_ev[2] = {nullptr, nullptr};  // lookahead round loop
  // stepwise driver state (vl_ransac_begin / step_score / step_finish / end)
  struct {
    Work wk;
    Inputs in;
    RansacParams p;
    int Q = 0, nactive = 0, open = 0;
    int64_t rounds = 0, max_rounds = 0;
  } step;
};

static void prof_hook(void* arg, int stage, bool begin) {
  vl_ctx* c = (vl_ctx*)arg;
  if (!c->prof) return;
  if (begin) {
    if (c->ev_used + 2 > c->ev_pool.size()) {
      for (int k = 0; k < 64; ++k) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->ev_pool.push_back(e);
      }
    }
    c->ev_stage.push_back(stage);
  }
  cudaEventRecord(c->ev_pool[c->ev_used++], c->prof_stream);
}

// Called after a stream sync: fold the recorded event pairs into the totals.
static void prof_collect(vl_ctx* c) {
  if (!c->prof) return;
  for (size_t i = 0; i < c->ev_stage.size(); ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]) == cudaSuccess) {
      c->stage_ms[c->ev_stage[i]] += ms;
      c->stage_launches[c->ev_stage[i]] += 1;
    }
  }
  c->ev_stage.clear();
  c->ev_used = 0;
}

static int fail(vl_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define VL_CUDA(ctx, expr)                                                                   \
  do {                                                                                       \
    cudaError_t e__ = (expr);                                                                \
    if (e__ != cudaSuccess)                                                                  \
      return fail(ctx, e__ == cudaErrorMemoryAllocation ? VL_ERR_OOM : VL_ERR_CUDA,          \
                  std::string(#expr) + ": " + cudaGetErrorString(e__));                     \
  } while (0)

static int ensure(vl_ctx* c, DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return VL_OK;
  if (b.p) {
    cudaError_t e = cudaFree(b.p);
    if (e != cudaSuccess) return fail(c, VL_ERR_CUDA, std::string("cudaFree: ") + cudaGetErrorString(e));
    b.p = nullptr;
    b.cap = 0;
  }
  size_t nb = bytes + bytes / 8;
  cudaError_t e = cudaMalloc(&b.p, nb);
  if (e != cudaSuccess) {
    b.p = nullptr;
    return fail(c, VL_ERR_OOM, "cudaMalloc(" + std::to_string(nb) + "): " + cudaGetErrorString(e));
  }
  b.cap = nb;
  return VL_OK;
}

// run totals of the pruning counters (evaluations skipped / evaluated by the
// scoring tail), zeroed when first allocated and by vl_scoring_counters
static int ensure_ctr(vl_ctx* c) {
  if (c->prune_ctr.p) return VL_OK;
  int rc = ensure(c, c->prune_ctr, 2 * sizeof(unsigned long long));
  if (rc) return rc;
  VL_CUDA(c, cudaMemset(c->prune_ctr.p, 0, 2 * sizeof(unsigned long long)));
  return VL_OK;
}

static int prune_enabled(vl_ctx* c) {
  if (c->prune < 0) {
    const char* e = getenv("VISLOC_PRUNE");
    c->prune = e ? (atoi(e) != 0) : 1;
  }
  return c->prune;
}

static int ensure_host(vl_ctx* c, size_t bytes) {
  if (c->h_pinned_cap >= bytes) return VL_OK;
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  c->h_pinned = nullptr;
  c->h_pinned_cap = 0;
  cudaError_t e = cudaMallocHost(&c->h_pinned, bytes);
  if (e != cudaSuccess) return fail(c, VL_ERR_OOM, std::string("cudaMallocHost: ") + cudaGetErrorString(e));
  c->h_pinned_cap = bytes;
  return VL_OK;
}

static int check_launch(vl_ctx* c) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, VL_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return VL_OK;
}

static GenState gen_from(const vl_pcg64_state& s) {
  GenState g;
  g.state = ((u128)s.state_hi << 64) | s.state_lo;
  g.inc = ((u128)s.inc_hi << 64) | s.inc_lo;
  g.has0 = s.has_uint32;
  g.uint0 = s.uinteger;
  return g;
}

static vl_pcg64_state state_from(const GenState& g) {
  vl_pcg64_state s;
  s.state_hi = (uint64_t)(g.state >> 64);
  s.state_lo = (uint64_t)g.state;
  s.inc_hi = (uint64_t)(g.inc >> 64);
  s.inc_lo = (uint64_t)g.inc;
  s.has_uint32 = g.has0;
  s.uinteger = g.uint0;
  return s;
}

// Generator state after `pos` 32-bit words were consumed (numpy semantics,
// including the stale `uinteger` value numpy reports).
static GenState advance_words(const GenState& g, uint64_t pos) {
  if (pos == 0) return g;
  GenState r = g;
  uint64_t k = pos;
  if (g.has0) k -= 1;  // the buffered word
  const uint64_t m = k >> 1;
  if ((k & 1) == 0) {
    r.state = pcg_advance(g.state, g.inc, m);
    r.has0 = 0;
    if (m > 0) r.uint0 = (uint32_t)(pcg_out(r.state) >> 32);
  } else {
    r.state = pcg_advance(g.state, g.inc, m + 1);
    r.has0 = 1;
    r.uint0 = (uint32_t)(pcg_out(r.state) >> 32);
  }
  return r;
}

extern "C" {

int vl_create(int device, vl_ctx** out) {
  if (!out) return VL_ERR_INVALID;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return VL_ERR_CUDA;
  if (device < 0 || device >= ndev) return VL_ERR_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return VL_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return VL_ERR_CUDA;
  if (prop.major != 10) return VL_ERR_CUDA;  // sm_100a build only
  vl_ctx* c = new vl_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  *out = c;
  return VL_OK;
}

int vl_destroy(vl_ctx* c) {
  if (!c) return VL_OK;
  cudaSetDevice(c->device);
  DevBuf* bufs[] = {&c->qs,      &c->active, &c->next_active, &c->active_count, &c->samples, &c->slots,
                    &c->slot_cnt, &c->p3p_geo, &c->p3p_cand, &c->p3p_nc, &c->P32, &c->P32s, &c->hsrc,        &c->items,        &c->item_count,
                    &c->partial, &c->cost32, &c->tile_cnt, &c->sub_pk, &c->sub32, &c->comp_pk,
                    &c->surv, &c->tail, &c->prune_ctr, &c->jump,
                    &c->samples2, &c->slots2, &c->slot_cnt2, &c->p3p_geo2, &c->p3p_cand2, &c->p3p_nc2,
                    &c->P32s2, &c->active2, &c->active_count2,
                    &c->scratch, &c->lift_meta, &c->lift_blk_count,
                    &c->lift_blk_off, &c->lift_seg_off, &c->tri_meta};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : c->round_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->pev)
    if (e) cudaEventDestroy(e);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  delete c;
  return VL_OK;
}

const char* vl_last_error(vl_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t vl_launch_count(vl_ctx* c) { return c ? c->launches : -1; }

int vl_profile(vl_ctx* c, int enable) {
  if (!c) return VL_ERR_INVALID;
  c->prof = enable ? 1 : 0;
  for (int k = 0; k < kNumStages; ++k) {
    c->stage_ms[k] = 0;
    c->stage_launches[k] = 0;
  }
  c->ev_stage.clear();
  c->ev_used = 0;
  return VL_OK;
}

int vl_profile_read(vl_ctx* c, double* ms, int64_t* launches, int32_t n) {
  if (!c || !ms || !launches) return VL_ERR_INVALID;
  for (int k = 0; k < n && k < kNumStages; ++k) {
    ms[k] = c->stage_ms[k];
    launches[k] = c->stage_launches[k];
  }
  return VL_OK;
}

int vl_set_scoring_pruning(vl_ctx* c, int32_t enable) {
  if (!c) return VL_ERR_INVALID;
  c->prune = enable ? 1 : 0;
  return VL_OK;
}

int vl_scoring_counters(vl_ctx* c, int64_t* out, int32_t reset) {
  if (!c || !out) return fail(c, VL_ERR_INVALID, "null argument");
  VL_CUDA(c, cudaSetDevice(c->device));
  int rc;
  if ((rc = ensure_ctr(c))) return rc;
  unsigned long long h[2];
  VL_CUDA(c, cudaDeviceSynchronize());
  VL_CUDA(c, cudaMemcpy(h, c->prune_ctr.p, sizeof h, cudaMemcpyDeviceToHost));
  out[0] = (int64_t)h[0];
  out[1] = (int64_t)h[1];
  if (reset) VL_CUDA(c, cudaMemset(c->prune_ctr.p, 0, sizeof h));
  return VL_OK;
}

int vl_pcg64_seed(uint64_t seed, vl_pcg64_state* out) {
  if (!out) return VL_ERR_INVALID;
  *out = state_from(seed_pcg64(seed));
  return VL_OK;
}

int vl_reserve(vl_ctx* c, int32_t max_queries, int64_t max_n_per_query, int32_t batch_size) {
  if (!c || max_queries <= 0 || max_n_per_query < 3 || batch_size <= 0) return VL_ERR_INVALID;
  cudaSetDevice(c->device);
  const int64_t Qc = max_queries, B = batch_size, H = 4 * B;
  const int64_t nsub = std::min<int64_t>(max_n_per_query, 10000);
  const int64_t ns = (nsub + kScoreChunk - 1) / kScoreChunk;
  int rc = VL_OK;
  rc |= ensure(c, c->samples, Qc * B * 3 * sizeof(int));
  rc |= ensure(c, c->slots, Qc * ((B + 31) / 32 * 32) * 48 * sizeof(double));
  rc |= ensure(c, c->slot_cnt, Qc * B * sizeof(int));
  const int64_t B32 = (B + 31) / 32 * 32;  // P3P scratch is blocked by 32 samples
  rc |= ensure(c, c->p3p_geo, Qc * B32 * kGeoDoubles * sizeof(double));
  rc |= ensure(c, c->p3p_cand, Qc * B32 * 3 * kMaxCandSlots * sizeof(double));
  rc |= ensure(c, c->p3p_nc, Qc * B * sizeof(int));
  rc |= ensure(c, c->P32, Qc * 12 * H * sizeof(float));
  rc |= ensure(c, c->P32s, Qc * 12 * H * sizeof(float));
  rc |= ensure(c, c->hsrc, Qc * H * sizeof(int));
  rc |= ensure(c, c->partial, Qc * ns * H * sizeof(float));
  rc |= ensure(c, c->cost32, Qc * H * sizeof(float));
  rc |= ensure(c, c->tile_cnt, Qc * ((H + kScoreTileHypsFine - 1) / kScoreTileHypsFine) * sizeof(int));
  return rc ? VL_ERR_OOM : VL_OK;
}

}  // extern "C"

// Validates the arguments and fills the round parameters.
static int ransac_params(vl_ctx* c, const vl_ransac_args* a, RansacParams& p) {
  const vl_ransac_config& cfg = a->cfg;
  if (!(cfg.reproj_threshold > 0)) return fail(c, VL_ERR_INVALID, "reproj_threshold must be positive");
  if (!(cfg.miss_probability > 0 && cfg.miss_probability < 1))
    return fail(c, VL_ERR_INVALID, "miss_probability must be in (0, 1)");
  if (cfg.batch_size <= 0 || cfg.batch_size > cfg.max_iterations)
    return fail(c, VL_ERR_INVALID, "batch_size must be in [1, max_iterations]");
  if (cfg.max_scoring <= 0 || cfg.lm_max_iters < 0) return fail(c, VL_ERR_INVALID, "bad config");
  const double cauchy = cfg.cauchy_scale > 0 ? cfg.cauchy_scale : cfg.reproj_threshold;
  const int Q = a->num_queries;
  if (Q <= 0) return fail(c, VL_ERR_INVALID, "num_queries must be positive");
  if (!a->offsets || !a->intr || !a->rng || !a->px || !a->X || !a->w)
    return fail(c, VL_ERR_INVALID, "null input array");
  for (int q = 0; q < Q; ++q) {
    const int64_t n = a->offsets[q + 1] - a->offsets[q];
    if (n < 3) return fail(c, VL_ERR_UNDERCONSTRAINED, "need >= 3 matches, got " + std::to_string(n));
    if (n > 0x7FFFFFFF) return fail(c, VL_ERR_INVALID, "more than 2^31-1 matches in one query");
  }
  p.max_iterations = cfg.max_iterations;
  p.batch_size = cfg.batch_size;
  p.lm_max_iters = cfg.lm_max_iters;
  p.eta = cfg.miss_probability;
  p.tau = cfg.reproj_threshold;
  p.cauchy = cauchy;
  return VL_OK;
}

// Largest query chunk whose per-round workspace stays bounded (~6 GB).
static int64_t ransac_chunk(int64_t Q, int64_t B) {
  const int64_t HCAP = 4 * B;
  const int64_t per_q = B * (3 * 4 + 48 * 8 + 4) + HCAP * (12 * 4 + 4) + HCAP * 4 * 20;
  int64_t Qc = std::max<int64_t>(1, std::min<int64_t>(Q, (int64_t)6e9 / per_q));
  return std::min<int64_t>(Qc, 4096);
}

// Uploads per-query state for queries [q0, q0+Qn), sizes the workspace and
// runs k_prep.  Fills `wk`.
static int setup_chunk(vl_ctx* c, const vl_ransac_args* a, int64_t q0, int Qn, const Inputs& in, Work& wk,
                       cudaStream_t st, QState** staged_qs = nullptr) {
  const vl_ransac_config& cfg = a->cfg;
  const int64_t B = cfg.batch_size;
  const int64_t HCAP = 4 * B;
  std::vector<QState> hq;
  {
    hq.assign(Qn, QState());
    int64_t nsub_tot = 0, ncomp = 0;
    int max_split = 1;
    for (int i = 0; i < Qn; ++i) {
      const int64_t gq = q0 + i;
      QState& S = hq[i];
      std::memset(&S, 0, sizeof(QState));
      const int64_t n = a->offsets[gq + 1] - a->offsets[gq];
      S.gen = gen_from(a->rng[gq]);
      S.off = a->offsets[gq];
      S.coff = ncomp;
      S.n = (int)n;
      S.stride = (int)((n + cfg.max_scoring - 1) / cfg.max_scoring);
      S.nsub = (int)((n + S.stride - 1) / S.stride);
      S.nsplit = (S.nsub + kScoreChunk - 1) / kScoreChunk;
      S.sub_off = nsub_tot;
      S.in = Intr{a->intr[gq].fx, a->intr[gq].fy, a->intr[gq].cx, a->intr[gq].cy};
      S.active = 1;
      S.best_cost = INFINITY;
      S.best.q[0] = 1.0;
      nsub_tot += S.nsub + (S.nsub & 1);  // even offsets: fp32 records are stored in pairs
      ncomp += n;
      max_split = std::max(max_split, S.nsplit);
    }
    // worst case: fine items (256-hypothesis tiles x 1 split)
    const int64_t ntile = (HCAP + kScoreTileHypsFine - 1) / kScoreTileHypsFine;
    const int64_t item_cap = (int64_t)Qn * ntile * max_split;
    int rc = VL_OK;
    if ((rc = ensure(c, c->qs, Qn * sizeof(QState))) ||
        (rc = ensure(c, c->active, Qn * sizeof(int))) ||
        (rc = ensure(c, c->active_count, 2 * sizeof(int))) ||
        (rc = ensure(c, c->samples, Qn * B * 3 * sizeof(int))) ||
        (rc = ensure(c, c->slots, Qn * ((B + 31) / 32 * 32) * 48 * sizeof(double))) ||
        (rc = ensure(c, c->slot_cnt, Qn * B * sizeof(int))) ||
        (rc = ensure(c, c->p3p_geo, Qn * ((B + 31) / 32 * 32) * kGeoDoubles * sizeof(double))) ||
        (rc = ensure(c, c->p3p_cand, Qn * ((B + 31) / 32 * 32) * 3 * kMaxCandSlots * sizeof(double))) ||
        (rc = ensure(c, c->p3p_nc, Qn * B * sizeof(int))) ||
        (rc = ensure(c, c->P32, Qn * 12 * HCAP * sizeof(float))) ||
        (rc = ensure(c, c->P32s, Qn * 12 * HCAP * sizeof(float))) ||
        (rc = ensure(c, c->hsrc, Qn * HCAP * sizeof(int))) ||
        (rc = ensure(c, c->items, item_cap * sizeof(ScoreItem))) ||
        (rc = ensure(c, c->item_count, 4 * sizeof(int))) ||
        (rc = ensure(c, c->partial, (size_t)Qn * max_split * HCAP * sizeof(float))) ||
        (rc = ensure(c, c->cost32, (size_t)Qn * HCAP * sizeof(float))) ||
        (rc = ensure(c, c->tile_cnt, (size_t)Qn * ntile * sizeof(int))) ||
        (rc = ensure(c, c->sub_pk, nsub_tot * 3 * sizeof(double2))) ||
        (rc = ensure(c, c->sub32, (nsub_tot / 2) * 3 * sizeof(float4))) ||
        (rc = ensure(c, c->comp_pk, ncomp * 3 * sizeof(double2))) ||
        (rc = ensure(c, c->surv, (size_t)Qn * HCAP * sizeof(int))) ||
        (rc = ensure(c, c->jump, (size_t)Qn * 2 * kJumpBits * sizeof(u128))) ||
        (rc = ensure(c, c->tail, (size_t)Qn * (HCAP / 32 + ntile) * sizeof(TailTask))) ||
        (rc = ensure_ctr(c)))
      return rc;
    const size_t host_bytes = Qn * sizeof(QState) + Qn * sizeof(int) + 64;
    if ((rc = ensure_host(c, host_bytes))) return rc;
    char* hp = (char*)c->h_pinned;
    QState* h_qs = (QState*)hp;
    // the pinned staging buffer is reused across chunks: previous copies finished at the last sync
    std::memcpy(h_qs, hq.data(), Qn * sizeof(QState));
    wk = Work();
    wk.qs = (QState*)c->qs.p;
    wk.active_list = (int*)c->active.p;
    wk.active_count = (int*)c->active_count.p;
    wk.next_active = nullptr;
    wk.samples = (int*)c->samples.p;
    wk.slots = (double*)c->slots.p;
    wk.slot_cnt = (int*)c->slot_cnt.p;
    wk.p3p_geo = (double*)c->p3p_geo.p;
    wk.p3p_cand = (double*)c->p3p_cand.p;
    wk.p3p_nc = (int*)c->p3p_nc.p;
    wk.P32 = (float*)c->P32.p;
    wk.P32s = (float*)c->P32s.p;
    wk.hsrc = (int*)c->hsrc.p;
    wk.items = (ScoreItem*)c->items.p;
    wk.item_count = (int*)c->item_count.p;
    wk.partial = (float*)c->partial.p;
    wk.cost32 = (float*)c->cost32.p;
    wk.tile_cnt = (int*)c->tile_cnt.p;
    wk.TCAP = (int)ntile;
    wk.sub_pk = (double2*)c->sub_pk.p;
    wk.sub32 = (float4*)c->sub32.p;
    wk.comp_pk = (double2*)c->comp_pk.p;
    wk.B = (int)B;
    wk.HCAP = (int)HCAP;
    wk.NSPLIT = max_split;
    wk.item_cap = item_cap;
    wk.split_rank = 0;
    wk.split_size = 1;
    wk.par = 0;
    wk.next_list = wk.active_list;
    wk.next_count = wk.active_count;
    wk.prune = prune_enabled(c);
    wk.jump = (u128*)c->jump.p;
    wk.surv = (int*)c->surv.p;
    wk.tail = (TailTask*)c->tail.p;
    wk.tail_cap = (int64_t)Qn * (HCAP / 32 + ntile);
    wk.prune_ctr = (unsigned long long*)c->prune_ctr.p;
    // k_prep pulls the states from the mapped staging buffer itself: no
    // copy-engine transfer on this stream (it would queue behind a concurrent
    // bulk host-to-device prefetch, see posest.ransac_pnp_host)
    QState* d_hqs = nullptr;
    VL_CUDA(c, cudaHostGetDevicePointer((void**)&d_hqs, h_qs, 0));
    VL_CUDA(c, cudaHostGetDevicePointer((void**)&wk.host_count,
                                        (char*)c->h_pinned + c->h_pinned_cap - 16, 0));
    c->prof_stream = st;
    if (staged_qs) {  // vl_ransac_pnp_staged admits the queries stage by stage
      *staged_qs = d_hqs;
      return VL_OK;
    }
    prof_hook(c, kStagePrep, true);
    c->launches += launch_prep(wk, in, 0, Qn, 0, d_hqs, st);
    prof_hook(c, kStagePrep, false);
    if ((rc = check_launch(c))) return rc;
  }
  return VL_OK;
}

// Reads back the active-query count after a round (the one host sync per round).
static int read_active(vl_ctx* c, const Work& wk, cudaStream_t st, int* nactive) {
  // k_scan's closing cluster mirrors the count into this mapped pinned word
  volatile int* h_count = (volatile int*)((char*)c->h_pinned + c->h_pinned_cap - 16);
  if (!wk.host_count) VL_CUDA(c, cudaMemcpyAsync((void*)h_count, wk.active_count, sizeof(int), cudaMemcpyDeviceToHost, st));
  VL_CUDA(c, cudaStreamSynchronize(st));
  prof_collect(c);
  *nactive = *h_count;
  return VL_OK;
}

extern "C" {

// Round loop with a one-round lookahead: round r+1 is queued (with the last
// count the host has read, a superset of the active queries; kernels skip list
// positions >= the device-side count) before the host waits for round r's
// count, so the GPU never idles while the host reads it and launches.  The
// round queued after the last one is a no-op.
static int round_loop_lookahead(vl_ctx* c, const Work& wk, const Inputs& in, const RansacParams& p, int Qn,
                                int64_t max_rounds, cudaStream_t st) {
  if (!c->round_ev[0]) {
    for (auto& e : c->round_ev) VL_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  volatile int* h_count = (volatile int*)((char*)c->h_pinned + c->h_pinned_cap - 16);
  int nlaunch = Qn;
  int64_t r = 0;
  // the first round splits (head / rest) for the queries that have no best pose yet
  c->launches += launch_round(wk, in, p, nlaunch, c->num_sms, st, nullptr, nullptr, 0, 1);
  VL_CUDA(c, cudaEventRecord(c->round_ev[0], st));
  while (true) {
    c->launches += launch_round(wk, in, p, nlaunch, c->num_sms, st, nullptr, nullptr, 0);
    int rc;
    if ((rc = check_launch(c))) return rc;
    VL_CUDA(c, cudaEventRecord(c->round_ev[(r + 1) & 1], st));
    VL_CUDA(c, cudaEventSynchronize(c->round_ev[r & 1]));  // round r (not the queued one) is done
    const int n = *h_count;  // the mirror of the count after round r (or a later round)
    if (n == 0) break;
    nlaunch = n;
    if (++r > max_rounds) return fail(c, VL_ERR_CUDA, "round loop did not terminate");
  }
  return VL_OK;
}

// Pipelined round loop for small batches (fine scoring rounds: the GPU is
// far from full): the side stream samples and solves P3P for round r+1 while
// the caller's stream scores and scans round r.  The sampler's outputs are
// double-buffered by round parity (Work::par), round r+1's side chain reads
// round r's active list (a superset: a query that stops after round r wastes
// one speculative batch, never its results — k_scan commits the iteration
// count), and k_scan compacts into the other list.  Same kernels, same
// arithmetic, identical results to round_loop_lookahead.
static bool pipeline_enabled() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("VISLOC_PIPE");
    mode = e ? (atoi(e) != 0) : 1;
  }
  return mode != 0;
}

static int round_loop_pipelined(vl_ctx* c, const Work& wk, const Inputs& in, const RansacParams& p, int Qn,
                                int64_t max_rounds, cudaStream_t st) {
  const int64_t B = wk.B, B32 = (B + 31) / 32 * 32, HCAP = wk.HCAP;
  int rc;
  if ((rc = ensure(c, c->samples2, Qn * B * 3 * sizeof(int))) ||
      (rc = ensure(c, c->slots2, Qn * B32 * 48 * sizeof(double))) ||
      (rc = ensure(c, c->slot_cnt2, Qn * B * sizeof(int))) ||
      (rc = ensure(c, c->p3p_geo2, Qn * B32 * kGeoDoubles * sizeof(double))) ||
      (rc = ensure(c, c->p3p_cand2, Qn * B32 * 3 * kMaxCandSlots * sizeof(double))) ||
      (rc = ensure(c, c->p3p_nc2, Qn * B * sizeof(int))) ||
      (rc = ensure(c, c->P32s2, Qn * 12 * HCAP * sizeof(float))) ||
      (rc = ensure(c, c->active2, Qn * sizeof(int))) || (rc = ensure(c, c->active_count2, 2 * sizeof(int))))
    return rc;
  if (!c->side) VL_CUDA(c, cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  if (!c->pev[0])
    for (auto& e : c->pev) VL_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (!c->round_ev[0])
    for (auto& e : c->round_ev) VL_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // main view of round r: W[r & 1] (its buffers, its list, compaction into the other list)
  Work W[2] = {wk, wk};
  W[1].par = 1;
  W[1].samples = (int*)c->samples2.p;
  W[1].slots = (double*)c->slots2.p;
  W[1].slot_cnt = (int*)c->slot_cnt2.p;
  W[1].p3p_geo = (double*)c->p3p_geo2.p;
  W[1].p3p_cand = (double*)c->p3p_cand2.p;
  W[1].p3p_nc = (int*)c->p3p_nc2.p;
  W[1].P32s = (float*)c->P32s2.p;
  W[1].active_list = (int*)c->active2.p;
  W[1].active_count = (int*)c->active_count2.p;
  W[0].next_list = W[1].active_list;
  W[0].next_count = W[1].active_count;
  W[1].next_list = W[0].active_list;
  W[1].next_count = W[0].active_count;
  // side view of round r: W[r & 1]'s buffers, the list of round r - 1 (round 0: the admitted list)
  auto side_view = [&](int64_t r) {
    Work v = W[r & 1];
    if (r > 0) {
      v.active_list = W[(r - 1) & 1].active_list;
      v.active_count = W[(r - 1) & 1].active_count;
    }
    return v;
  };
  cudaEvent_t ev_start = c->pev[0], ev_p[2] = {c->pev[1], c->pev[2]}, ev_c[2] = {c->pev[3], c->pev[4]};
  cudaEvent_t ev_end = c->pev[5];
  volatile int* h_count = (volatile int*)((char*)c->h_pinned + c->h_pinned_cap - 16);
  VL_CUDA(c, cudaEventRecord(ev_start, st));  // the admitted queries (k_prep)
  VL_CUDA(c, cudaStreamWaitEvent(c->side, ev_start, 0));
  c->launches += launch_round(side_view(0), in, p, Qn, c->num_sms, c->side, nullptr, nullptr, 3);
  VL_CUDA(c, cudaEventRecord(ev_p[0], c->side));
  int nlaunch = Qn;
  // queue round r: compaction (after its side chain), round r+1's side chain
  // (after the compaction: it overwrites round r-1's buffers), scores + scan
  auto queue = [&](int64_t r) -> int {
    VL_CUDA(c, cudaStreamWaitEvent(st, ev_p[r & 1], 0));
    c->launches += launch_round(W[r & 1], in, p, nlaunch, c->num_sms, st, nullptr, nullptr, 4);
    VL_CUDA(c, cudaEventRecord(ev_c[r & 1], st));
    VL_CUDA(c, cudaStreamWaitEvent(c->side, ev_c[r & 1], 0));
    c->launches += launch_round(side_view(r + 1), in, p, nlaunch, c->num_sms, c->side, nullptr, nullptr, 3);
    VL_CUDA(c, cudaEventRecord(ev_p[(r + 1) & 1], c->side));
    c->launches += launch_round(W[r & 1], in, p, nlaunch, c->num_sms, st, nullptr, nullptr, 5);
    VL_CUDA(c, cudaEventRecord(c->round_ev[r & 1], st));
    return check_launch(c);
  };
  int64_t r = 0;
  if ((rc = queue(0))) return rc;
  while (true) {
    if ((rc = queue(r + 1))) return rc;  // one round ahead, with the last count read (a superset)
    VL_CUDA(c, cudaEventSynchronize(c->round_ev[r & 1]));
    const int n = *h_count;
    if (n == 0) break;
    nlaunch = n;
    if (++r > max_rounds) return fail(c, VL_ERR_CUDA, "round loop did not terminate");
  }
  // the side stream's queued speculative work ends before anything reuses its buffers
  VL_CUDA(c, cudaEventRecord(ev_end, c->side));
  VL_CUDA(c, cudaStreamWaitEvent(st, ev_end, 0));
  return VL_OK;
}

int vl_ransac_pnp(vl_ctx* c, const vl_ransac_args* a, const vl_ransac_out* o, void* stream) {
  if (!c || !a || !o) return fail(c, VL_ERR_INVALID, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  RansacParams p;
  int rc;
  if ((rc = ransac_params(c, a, p))) return rc;
  VL_CUDA(c, cudaSetDevice(c->device));
  const int Q = a->num_queries;
  const int64_t B = a->cfg.batch_size;
  const int64_t Qc = ransac_chunk(Q, B);
  Inputs in{a->px, a->X, a->w};
  Outputs out{o->q, o->t, o->inlier_flags, o->inlier_count, o->score, o->iterations, o->converged, o->stats};
  const int64_t max_rounds = (a->cfg.max_iterations + B - 1) / B + 1;
  for (int64_t q0 = 0; q0 < Q; q0 += Qc) {
    const int Qn = (int)std::min<int64_t>(Qc, Q - q0);
    Work wk;
    if ((rc = setup_chunk(c, a, q0, Qn, in, wk, st))) return rc;
    int nactive = Qn;
    int guard = 0;
    if (c->prof) {  // per-stage event brackets: one round in flight at a time
      while (nactive > 0) {
        c->launches += launch_round(wk, in, p, nactive, c->num_sms, st, prof_hook, c, 0, guard == 0);
        if ((rc = check_launch(c))) return rc;
        if ((rc = read_active(c, wk, st, &nactive))) return rc;
        if (++guard > max_rounds) return fail(c, VL_ERR_CUDA, "round loop did not terminate");
      }
    } else if (pipeline_enabled() && round_is_fine(wk, Qn, c->num_sms)) {
      if ((rc = round_loop_pipelined(c, wk, in, p, Qn, max_rounds, st))) return rc;
    } else if ((rc = round_loop_lookahead(c, wk, in, p, Qn, max_rounds, st))) {
      return rc;
    }
    prof_hook(c, kStageFinal, true);
    c->launches += launch_final(wk, in, out, p, Qn, (int)q0, st);
    prof_hook(c, kStageFinal, false);
    if ((rc = check_launch(c))) return rc;
    if (q0 + Qc < Q || c->prof) {
      VL_CUDA(c, cudaStreamSynchronize(st));  // staging buffer reuse / event readout
      prof_collect(c);
    }
  }
  return VL_OK;
}

// ---- staged admission (host pipeline) --------------------------------------
// Queries of stage k ([stage_end[k-1], stage_end[k])) join the running round
// loop as soon as their input copy (event k) has completed; the first stage
// is waited for on the stream.  One estimator run over all queries, so the
// host-to-device copy of later stages overlaps the rounds of earlier ones
// without the tail cost of separate per-chunk runs.  Per-query results are
// identical to vl_ransac_pnp (each query's computation is independent of
// which others share its rounds).
// One workspace chunk [q0, q0 + Qn) of a staged run; `ends` (chunk-relative)
// and `evs` are the stages clipped to the chunk.
static int staged_chunk(vl_ctx* c, const vl_ransac_args* a, int64_t q0, int Qn, const std::vector<int>& ends,
                        const std::vector<cudaEvent_t>& evs, const Inputs& in, const Outputs& out,
                        const RansacParams& p, cudaStream_t st) {
  const int64_t B = a->cfg.batch_size;
  const int nstage = (int)ends.size();
  Work wk;
  QState* d_hqs = nullptr;
  int rc;
  if ((rc = setup_chunk(c, a, q0, Qn, in, wk, st, &d_hqs))) return rc;
  const int64_t max_rounds = ((a->cfg.max_iterations + B - 1) / B + 1) * (int64_t)nstage + nstage;
  int admitted = 0, nactive = 0, guard = 0;
  while (true) {
    // admit every stage whose copy has landed (block on the next one only when idle)
    const int admitted0 = admitted;
    while (admitted < nstage) {
      cudaEvent_t ev = evs[admitted];
      if (nactive > 0) {
        const cudaError_t e = cudaEventQuery(ev);
        if (e == cudaErrorNotReady) break;
        if (e != cudaSuccess) return fail(c, VL_ERR_CUDA, std::string("cudaEventQuery: ") + cudaGetErrorString(e));
      }
      VL_CUDA(c, cudaStreamWaitEvent(st, ev, 0));
      const int s0 = admitted ? ends[admitted - 1] : 0, s1 = ends[admitted];
      prof_hook(c, kStagePrep, true);
      c->launches += launch_prep(wk, in, s0, s1 - s0, nactive, d_hqs, st);
      prof_hook(c, kStagePrep, false);
      if ((rc = check_launch(c))) return rc;
      nactive += s1 - s0;
      ++admitted;
    }
    if (nactive == 0) break;
    if (admitted == nstage && !c->prof) {  // everything admitted: finish with the lookahead loop
      if ((rc = round_loop_lookahead(c, wk, in, p, nactive, max_rounds, st))) return rc;
      break;
    }
    // (a round right after an admission splits for the new queries)
    c->launches += launch_round(wk, in, p, nactive, c->num_sms, st, prof_hook, c, 0, admitted > admitted0);
    if ((rc = check_launch(c))) return rc;
    if ((rc = read_active(c, wk, st, &nactive))) return rc;
    if (++guard > max_rounds) return fail(c, VL_ERR_CUDA, "round loop did not terminate");
  }
  prof_hook(c, kStageFinal, true);
  c->launches += launch_final(wk, in, out, p, Qn, (int)q0, st);
  prof_hook(c, kStageFinal, false);
  return check_launch(c);
}

int vl_ransac_pnp_staged(vl_ctx* c, const vl_ransac_args* a, const vl_ransac_out* o, int32_t nstage,
                         const int32_t* stage_end, void* const* stage_events, void* stream) {
  if (!c || !a || !o || nstage < 1 || !stage_end || !stage_events) return fail(c, VL_ERR_INVALID, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  RansacParams p;
  int rc;
  if ((rc = ransac_params(c, a, p))) return rc;
  const int Q = a->num_queries;
  for (int k = 0; k < nstage; ++k)
    if (stage_end[k] <= (k ? stage_end[k - 1] : 0) || !stage_events[k])
      return fail(c, VL_ERR_INVALID, "stages must be non-empty, increasing, with an event each");
  if (stage_end[nstage - 1] != Q) return fail(c, VL_ERR_INVALID, "last stage must end at num_queries");
  VL_CUDA(c, cudaSetDevice(c->device));
  Inputs in{a->px, a->X, a->w};
  Outputs out{o->q, o->t, o->inlier_flags, o->inlier_count, o->score, o->iterations, o->converged, o->stats};
  // a run larger than one workspace chunk: the chunks run one after another,
  // each admitting the stages that overlap it as their copies land
  const int64_t Qc = ransac_chunk(Q, a->cfg.batch_size);
  for (int64_t q0 = 0; q0 < Q; q0 += Qc) {
    const int Qn = (int)std::min<int64_t>(Qc, Q - q0);
    std::vector<int> ends;
    std::vector<cudaEvent_t> evs;
    for (int k = 0; k < nstage; ++k) {
      const int64_t lo = std::max<int64_t>(k ? stage_end[k - 1] : 0, q0);
      const int64_t hi = std::min<int64_t>(stage_end[k], q0 + Qn);
      if (lo < hi) {
        ends.push_back((int)(hi - q0));
        evs.push_back((cudaEvent_t)stage_events[k]);
      }
    }
    if ((rc = staged_chunk(c, a, q0, Qn, ends, evs, in, out, p, st))) return rc;
    if (q0 + Qc < Q || c->prof) {
      VL_CUDA(c, cudaStreamSynchronize(st));  // staging buffer reuse / event readout
      prof_collect(c);
    }
  }
  return VL_OK;
}

// ---- stepwise driver (hypothesis-split mode) ------------------
// Every rank runs the same queries with the same seeds (identical samples,
// P3P and scans); the scoring tiles (query, 256/768 hypotheses) are dealt
// round-robin to ranks, the owner computes a tile's final fp32 costs and the
// other ranks hold zeros, so a SUM all-reduce of the [Q][HCAP] fp32 cost
// vector (x + 0 = x exactly) between vl_ransac_step_score and
// vl_ransac_step_finish gives every rank bit-identical costs — and the same
// final estimate as the single-GPU path.
int vl_ransac_begin(vl_ctx* c, const vl_ransac_args* a, int32_t split_rank, int32_t split_size, void* stream) {
  if (!c || !a) return fail(c, VL_ERR_INVALID, "null argument");
  if (split_size < 1 || split_rank < 0 || split_rank >= split_size) return fail(c, VL_ERR_INVALID, "bad split");
  RansacParams p;
  int rc;
  if ((rc = ransac_params(c, a, p))) return rc;
  if (ransac_chunk(a->num_queries, a->cfg.batch_size) < a->num_queries)
    return fail(c, VL_ERR_INVALID, "stepwise driver takes one workspace chunk of queries");
  VL_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  c->step.in = Inputs{a->px, a->X, a->w};
  if ((rc = setup_chunk(c, a, 0, a->num_queries, c->step.in, c->step.wk, st))) return rc;
  c->step.wk.split_rank = split_rank;
  c->step.wk.split_size = split_size;
  c->step.wk.prune = 0;  // the exchanged cost vectors are full costs (SUM / packed-argmin reductions)
  c->step.p = p;
  c->step.Q = a->num_queries;
  c->step.nactive = a->num_queries;
  c->step.rounds = 0;
  c->step.max_rounds = (a->cfg.max_iterations + a->cfg.batch_size - 1) / a->cfg.batch_size + 1;
  c->step.open = 1;
  return VL_OK;
}

int vl_ransac_partial_bytes(vl_ctx* c, int64_t* bytes) {
  if (!c || !c->step.open || !bytes) return fail(c, VL_ERR_INVALID, "no open stepwise run");
  *bytes = (int64_t)c->step.Q * c->step.wk.HCAP * (int64_t)sizeof(float);
  return VL_OK;
}

int vl_ransac_step_score(vl_ctx* c, void* partial_out, void* stream) {
  if (!c || !c->step.open) return fail(c, VL_ERR_INVALID, "no open stepwise run");
  cudaStream_t st = (cudaStream_t)stream;
  if (c->step.nactive <= 0) return fail(c, VL_ERR_INVALID, "no active queries");
  c->launches += launch_round(c->step.wk, c->step.in, c->step.p, c->step.nactive, c->num_sms, st, prof_hook, c, 1);
  int rc;
  if ((rc = check_launch(c))) return rc;
  if (partial_out) {
    const size_t bytes = (size_t)c->step.Q * c->step.wk.HCAP * sizeof(float);
    VL_CUDA(c, cudaMemcpyAsync(partial_out, c->step.wk.cost32, bytes, cudaMemcpyDeviceToDevice, st));
  }
  return VL_OK;
}

int vl_ransac_step_finish(vl_ctx* c, const void* partial_in, int32_t* nactive, void* stream) {
  if (!c || !c->step.open || !nactive) return fail(c, VL_ERR_INVALID, "no open stepwise run");
  cudaStream_t st = (cudaStream_t)stream;
  if (partial_in) {
    const size_t bytes = (size_t)c->step.Q * c->step.wk.HCAP * sizeof(float);
    VL_CUDA(c, cudaMemcpyAsync(c->step.wk.cost32, partial_in, bytes, cudaMemcpyDeviceToDevice, st));
  }
  c->launches += launch_round(c->step.wk, c->step.in, c->step.p, c->step.nactive, c->num_sms, st, prof_hook, c, 2);
  int rc;
  if ((rc = check_launch(c))) return rc;
  int na = 0;
  if ((rc = read_active(c, c->step.wk, st, &na))) return rc;
  c->step.nactive = na;
  *nactive = na;
  if (++c->step.rounds > c->step.max_rounds) return fail(c, VL_ERR_CUDA, "round loop did not terminate");
  return VL_OK;
}

int vl_ransac_step_argmin(vl_ctx* c, int64_t* keys, void* stream) {
  if (!c || !c->step.open || !keys) return fail(c, VL_ERR_INVALID, "no open stepwise run");
  if (c->step.nactive <= 0) return fail(c, VL_ERR_INVALID, "no active queries");
  cudaStream_t st = (cudaStream_t)stream;
  c->launches += launch_fill_i64((long long*)keys, c->step.Q, INT64_MAX, st);  // inactive queries: no candidate
  c->launches += launch_split_argmin(c->step.wk, c->step.nactive, c->num_sms, (long long*)keys, st);
  return check_launch(c);
}

int vl_ransac_step_finish_argmin(vl_ctx* c, const int64_t* keys, int32_t* nactive, void* stream) {
  if (!c || !c->step.open || !keys || !nactive) return fail(c, VL_ERR_INVALID, "no open stepwise run");
  cudaStream_t st = (cudaStream_t)stream;
  c->launches += launch_split_apply_argmin(c->step.wk, c->step.nactive, (const long long*)keys, st);
  int rc;
  if ((rc = check_launch(c))) return rc;
  return vl_ransac_step_finish(c, nullptr, nactive, stream);
}

int vl_ransac_end(vl_ctx* c, const vl_ransac_out* o, void* stream) {
  if (!c || !c->step.open || !o) return fail(c, VL_ERR_INVALID, "no open stepwise run");
  if (c->step.nactive != 0) return fail(c, VL_ERR_INVALID, "queries still active");
  cudaStream_t st = (cudaStream_t)stream;
  Outputs out{o->q, o->t, o->inlier_flags, o->inlier_count, o->score, o->iterations, o->converged, o->stats};
  c->launches += launch_final(c->step.wk, c->step.in, out, c->step.p, c->step.Q, 0, st);
  c->step.open = 0;
  return check_launch(c);
}

static Pose pose_from_host(const double* q, const double* t) {
  Pose p;
  for (int i = 0; i < 4; ++i) p.q[i] = q[i];
  for (int i = 0; i < 3; ++i) p.t[i] = t[i];
  return p;
}

int vl_msac_score(vl_ctx* c, const double* q, const double* t, const double* px, const double* X,
                  const double* w, int64_t n, vl_intrinsics intr, double tau, double* cost_out,
                  uint8_t* flags, void* stream) {
  if (!c || !q || !t || !cost_out || n < 0) return fail(c, VL_ERR_INVALID, "bad argument");
  if (n > 0x7FFFFFFF) return fail(c, VL_ERR_INVALID, "n too large");
  VL_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = ensure(c, c->scratch, 4096))) return rc;
  if ((rc = ensure_host(c, 4096))) return rc;
  double* dred = (double*)c->scratch.p;
  c->launches += launch_msac(pose_from_host(q, t), px, X, w, (int)n, Intr{intr.fx, intr.fy, intr.cx, intr.cy},
                             tau, dred, flags, st);
  if ((rc = check_launch(c))) return rc;
  double* h = (double*)c->h_pinned;
  VL_CUDA(c, cudaMemcpyAsync(h, dred, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  VL_CUDA(c, cudaStreamSynchronize(st));
  *cost_out = h[0];
  return VL_OK;
}

int vl_score_hypotheses(vl_ctx* c, const double* R, const double* t, int32_t H, const double* px,
                        const double* X, const double* w, int64_t n, vl_intrinsics intr, double tau,
                        int32_t shape, float* costs, void* stream) {
  if (!c || !R || !t || !px || !X || !w || !costs || H < 0 || n < 1 || shape < 0 || shape > 2)
    return fail(c, VL_ERR_INVALID, "bad argument");
  if (!(tau > 0)) return fail(c, VL_ERR_INVALID, "tau must be positive");
  if (n > 0x7FFFFFFF || H > (1 << 28)) return fail(c, VL_ERR_INVALID, "n or H too large");
  // it scores in the estimator's workspace: not while a stepwise run holds it
  if (c->step.open) return fail(c, VL_ERR_INVALID, "context has an open stepwise run (vl_ransac_begin)");
  if (H == 0) return VL_OK;
  VL_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  QState S;
  std::memset(&S, 0, sizeof(QState));
  S.n = S.nsub = (int)n;
  S.stride = 1;
  S.nsplit = (int)((n + kScoreChunk - 1) / kScoreChunk);
  S.in = Intr{intr.fx, intr.fy, intr.cx, intr.cy};
  S.nh = H;
  S.h_lo = 0;
  S.h_hi = H;
  // tile shape: the one the estimator picks for a lone query (fine), or forced
  const int fine = shape == 2 ? 0 : 1;
  const int64_t HCAP = H, ntile = (H + kScoreTileHypsFine - 1) / kScoreTileHypsFine;
  const int64_t nsub_pad = n + (n & 1);
  int rc;
  if ((rc = ensure(c, c->qs, sizeof(QState))) || (rc = ensure(c, c->items, ntile * S.nsplit * sizeof(ScoreItem))) ||
      (rc = ensure(c, c->item_count, 4 * sizeof(int))) || (rc = ensure(c, c->P32, 12 * HCAP * sizeof(float))) ||
      (rc = ensure(c, c->hsrc, HCAP * sizeof(int))) ||
      (rc = ensure(c, c->partial, (size_t)S.nsplit * HCAP * sizeof(float))) ||
      (rc = ensure(c, c->cost32, HCAP * sizeof(float))) || (rc = ensure(c, c->tile_cnt, ntile * sizeof(int))) ||
      (rc = ensure(c, c->sub_pk, nsub_pad * 3 * sizeof(double2))) ||
      (rc = ensure(c, c->sub32, (nsub_pad / 2) * 3 * sizeof(float4))))
    return rc;
  Work wk{};
  wk.prune = 0;  // every hypothesis' full cost is the output
  wk.qs = (QState*)c->qs.p;
  wk.items = (ScoreItem*)c->items.p;
  wk.item_count = (int*)c->item_count.p;
  wk.P32 = (float*)c->P32.p;
  wk.hsrc = (int*)c->hsrc.p;
  wk.partial = (float*)c->partial.p;
  wk.cost32 = (float*)c->cost32.p;
  wk.tile_cnt = (int*)c->tile_cnt.p;
  wk.sub_pk = (double2*)c->sub_pk.p;
  wk.sub32 = (float4*)c->sub32.p;
  wk.HCAP = (int)HCAP;
  wk.TCAP = (int)ntile;
  wk.NSPLIT = S.nsplit;
  wk.item_cap = ntile * S.nsplit;
  wk.split_rank = 0;
  wk.split_size = 1;
  VL_CUDA(c, cudaMemcpyAsync(wk.qs, &S, sizeof(QState), cudaMemcpyHostToDevice, st));
  Inputs in{px, X, w};
  c->launches += launch_prep(wk, in, 0, 1, 0, nullptr, st);  // scoring records, as every round reads them
  c->launches += launch_hyp_rows(wk, R, t, H, fine, st);
  c->launches += launch_score(wk, (float)(tau * tau), c->num_sms, fine, 1, st);
  if ((rc = check_launch(c))) return rc;
  VL_CUDA(c, cudaMemcpyAsync(costs, wk.cost32, H * sizeof(float), cudaMemcpyDeviceToDevice, st));
  VL_CUDA(c, cudaStreamSynchronize(st));  // the host-side state above is stack memory
  return VL_OK;
}

int vl_refine_pose(vl_ctx* c, double* q_io, double* t_io, const double* px, const double* X, const double* w,
                   int64_t n, vl_intrinsics intr, int32_t loss, double scale, int32_t max_iters,
                   double gradient_tol, double cost_tol, int32_t* converged, int32_t* iterations,
                   double* trace, int32_t* trace_len, void* stream) {
  if (!c || !q_io || !t_io || max_iters < 0 || (loss != 0 && loss != 1))
    return fail(c, VL_ERR_INVALID, "bad argument");
  if (!(scale > 0)) return fail(c, VL_ERR_INVALID, "scale must be positive");
  if (n < 3) return fail(c, VL_ERR_SINGULAR, "refinement needs >= 3 matches, got " + std::to_string(n));
  if (n > 0x7FFFFFFF) return fail(c, VL_ERR_INVALID, "n too large");
  VL_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t trace_bytes = (size_t)(max_iters + 1) * sizeof(double);
  const size_t need = 256 + trace_bytes;
  int rc;
  if ((rc = ensure(c, c->scratch, need))) return rc;
  if ((rc = ensure_host(c, need))) return rc;
  char* base = (char*)c->scratch.p;
  Pose* dpose = (Pose*)base;
  int* dinfo = (int*)(base + 128);
  double* dtrace = (double*)(base + 256);
  c->launches += launch_refine(pose_from_host(q_io, t_io), px, X, w, (int)n,
                               Intr{intr.fx, intr.fy, intr.cx, intr.cy}, loss, scale, max_iters, gradient_tol,
                               cost_tol, dpose, dinfo, dtrace, st);
  if ((rc = check_launch(c))) return rc;
  char* h = (char*)c->h_pinned;
  VL_CUDA(c, cudaMemcpyAsync(h, base, need, cudaMemcpyDeviceToHost, st));
  VL_CUDA(c, cudaStreamSynchronize(st));
  const Pose* hp = (const Pose*)h;
  const int* hi = (const int*)(h + 128);
  for (int i = 0; i < 4; ++i) q_io[i] = hp->q[i];
  for (int i = 0; i < 3; ++i) t_io[i] = hp->t[i];
  if (converged) *converged = hi[0];
  if (iterations) *iterations = hi[1];
  if (trace_len) *trace_len = hi[2];
  if (trace) std::memcpy(trace, h + 256, (size_t)hi[2] * sizeof(double));
  return VL_OK;
}

int vl_p3p_solve_batch(vl_ctx* c, const double* bearings, const double* points, int32_t B, double* R,
                       double* t, int64_t* sample, int32_t* m_out, void* stream) {
  if (!c || B < 0 || !m_out) return fail(c, VL_ERR_INVALID, "bad argument");
  *m_out = 0;
  if (B == 0) return VL_OK;
  VL_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = ensure(c, c->slots, (size_t)B * 48 * sizeof(double)))) return rc;
  if ((rc = ensure(c, c->slot_cnt, (size_t)B * sizeof(int) + 16))) return rc;
  if ((rc = ensure_host(c, 64))) return rc;
  int* dm = (int*)c->slot_cnt.p + B;
  c->launches += launch_p3p_batch(bearings, points, B, (double*)c->slots.p, (int*)c->slot_cnt.p, R, t, sample,
                                  dm, st);
  if ((rc = check_launch(c))) return rc;
  int* h = (int*)c->h_pinned;
  VL_CUDA(c, cudaMemcpyAsync(h, dm, sizeof(int), cudaMemcpyDeviceToHost, st));
  VL_CUDA(c, cudaStreamSynchronize(st));
  *m_out = *h;
  return VL_OK;
}

int vl_sample_minimal_sets(vl_ctx* c, vl_pcg64_state* stt, int64_t n, int32_t count, int32_t* out,
                           void* stream) {
  if (!c || !stt || count < 0) return fail(c, VL_ERR_INVALID, "bad argument");
  if (n < 3 || n > 0xFFFFFFFFll) return fail(c, VL_ERR_INVALID, "population must be in [3, 2^32)");
  if (count == 0) return VL_OK;
  VL_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = ensure(c, c->scratch, 64))) return rc;
  if ((rc = ensure_host(c, 64))) return rc;
  const GenState g = gen_from(*stt);
  uint64_t* dpos = (uint64_t*)c->scratch.p;
  c->launches += launch_sample(g, 0, n, count, out, dpos, st);
  if ((rc = check_launch(c))) return rc;
  uint64_t* h = (uint64_t*)c->h_pinned;
  VL_CUDA(c, cudaMemcpyAsync(h, dpos, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  VL_CUDA(c, cudaStreamSynchronize(st));
  *stt = state_from(advance_words(g, *h));
  return VL_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ lifting
#include "vl_lift.h"
static_assert(sizeof(vl_lift_segment) == sizeof(vl::LiftSeg), "segment layout");
static_assert(sizeof(vl_lift_depth) == sizeof(vl::LiftDepth), "depth layout");


extern "C" int vl_lift(vl_ctx* c, const vl_lift_segment* segs, int32_t nseg, const vl_lift_depth* depths,
                       int32_t ndepth, int32_t field_f64, double threshold, int32_t mode, double* px_out,
                       double* X_out, double* w_out, int32_t* entry_out, int64_t capacity,
                       int64_t* seg_offsets, int32_t* seg_flags, void* stream) {
  if (!c || nseg < 0 || (nseg > 0 && !segs) || !seg_offsets || (mode != 0 && mode != 1))
    return fail(c, VL_ERR_INVALID, "bad argument");
  if (!(threshold >= 0 && threshold <= 1))
    return fail(c, VL_ERR_INVALID, "threshold must be in [0, 1], got " + std::to_string(threshold));
  seg_offsets[0] = 0;
  if (nseg == 0) return VL_OK;
  VL_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t BC = lift_block_cells();
  std::vector<int64_t> blk0(nseg);
  int64_t nblk = 0;
  for (int s = 0; s < nseg; ++s) {
    const vl_lift_segment& S = segs[s];
    if (S.grid_w <= 0 || S.grid_h <= 0 || !S.targets || (S.layout == VL_LIFT_PLANAR && !S.confidence))
      return fail(c, VL_ERR_INVALID, "segment " + std::to_string(s) + ": empty grid or null arrays");
    if (S.layout != VL_LIFT_PLANAR && S.layout != VL_LIFT_IMLC)
      return fail(c, VL_ERR_INVALID, "segment " + std::to_string(s) + ": bad layout");
    if (S.layout == VL_LIFT_IMLC && ((uintptr_t)S.targets & 3))
      return fail(c, VL_ERR_INVALID, "segment " + std::to_string(s) + ": IMLC records must be 4-byte aligned");
    if ((int64_t)S.grid_w * S.grid_h > INT32_MAX)
      return fail(c, VL_ERR_INVALID, "segment " + std::to_string(s) + ": grid too large");
    if (mode == 0 && (S.depth < 0 || S.depth >= ndepth))
      return fail(c, VL_ERR_INVALID, "segment " + std::to_string(s) + ": bad depth index");
    if (S.direction != 0 && S.direction != 1) return fail(c, VL_ERR_INVALID, "bad direction");
    blk0[s] = nblk;
    nblk += ((int64_t)S.grid_w * S.grid_h + BC - 1) / BC;
  }
  if (mode == 0)
    for (int d = 0; d < ndepth; ++d) {
      const vl_lift_depth& D = depths[d];
      if (D.width < 2 || D.height < 2 || !D.values || (D.kind < 2 && !D.valid) || (D.kind >= 2 && !D.lut))
        return fail(c, VL_ERR_INVALID, "depth " + std::to_string(d) + ": bad map");
    }
  const size_t seg_bytes = nseg * sizeof(vl_lift_segment), dep_bytes = (mode == 0 ? ndepth : 0) * sizeof(vl_lift_depth);
  const size_t sob_bytes = ((size_t)nblk * sizeof(int) + 7) & ~(size_t)7;  // tile -> segment table
  const size_t meta = seg_bytes + dep_bytes + nseg * sizeof(int64_t) + sob_bytes;  // all multiples of 8
  // zeroed by k_lift_prep: seg_flags [nseg] int, the scan's ticket
  const size_t zflags = meta, zend = zflags + (size_t)(nseg + 1) * sizeof(int);
  const int64_t nchunk = (nblk + 1023) / 1024;
  const size_t host_bytes = meta + (nseg + 1) * sizeof(int64_t) + nseg * sizeof(int) + 64;
  int rc;
  if ((rc = ensure(c, c->lift_meta, zend)) || (rc = ensure(c, c->lift_blk_count, nblk * 9 * sizeof(int))) ||
      (rc = ensure(c, c->lift_blk_off, (nblk + nchunk) * sizeof(int64_t))) || (rc = ensure(c, c->lift_seg_off, (nseg + 1) * sizeof(int64_t))) ||
      (rc = ensure_host(c, host_bytes)))
    return rc;
  char* h = (char*)c->h_pinned;
  std::memcpy(h, segs, seg_bytes);
  if (dep_bytes) std::memcpy(h + seg_bytes, depths, dep_bytes);
  std::memcpy(h + seg_bytes + dep_bytes, blk0.data(), nseg * sizeof(int64_t));
  {
    int* sob = (int*)(h + seg_bytes + dep_bytes + nseg * sizeof(int64_t));
    for (int s = 0; s < nseg; ++s) {
      const int64_t e = s + 1 < nseg ? blk0[s + 1] : nblk;
      for (int64_t k = blk0[s]; k < e; ++k) sob[k] = s;
    }
  }
  char* d = (char*)c->lift_meta.p;
  int64_t* hoff = (int64_t*)(h + meta);
  int* hflags = (int*)(h + meta + (nseg + 1) * sizeof(int64_t));
  void *d_h = nullptr, *d_hoff = nullptr, *d_hflags = nullptr;
  VL_CUDA(c, cudaHostGetDevicePointer(&d_h, h, 0));
  VL_CUDA(c, cudaHostGetDevicePointer(&d_hoff, hoff, 0));
  VL_CUDA(c, cudaHostGetDevicePointer(&d_hflags, hflags, 0));
  // metadata pulled by a kernel from mapped pinned memory and results pushed
  // back the same way: no copy-engine transfers queued on this stream
  c->launches += launch_lift_prep(d, d_h, meta, (int*)(d + zflags), (int)((zend - zflags) / sizeof(int)), st);
  LiftArgs a;
  a.segs = (const LiftSeg*)d;
  a.nseg = nseg;
  a.depths = (const LiftDepth*)(d + seg_bytes);
  a.seg_blk0 = (const int64_t*)(d + seg_bytes + dep_bytes);
  a.seg_of_blk = (const int*)(d + seg_bytes + dep_bytes + nseg * sizeof(int64_t));
  a.nblk = nblk;
  a.blk_count = (int*)c->lift_blk_count.p;
  a.warp_count = a.blk_count + nblk;
  a.blk_off = (int64_t*)c->lift_blk_off.p;
  a.seg_off = (int64_t*)c->lift_seg_off.p;
  a.seg_flags = (int*)(d + zflags);
  a.scan_ticket = (int*)(d + zflags) + nseg;
  a.chunk_off = (int64_t*)c->lift_blk_off.p + nblk;
  a.seg_off_host = (int64_t*)d_hoff;
  a.seg_flags_host = (int*)d_hflags;
  a.threshold = threshold;
  a.px_out = px_out;
  a.X_out = X_out;
  a.w_out = w_out;
  a.entry_out = entry_out;
  a.capacity = capacity;
  c->prof_stream = st;
  prof_hook(c, kStageLift, true);
  c->launches += launch_lift(a, field_f64, mode, st);
  prof_hook(c, kStageLift, false);
  if ((rc = check_launch(c))) return rc;
  VL_CUDA(c, cudaStreamSynchronize(st));
  std::memcpy(seg_offsets, hoff, (nseg + 1) * sizeof(int64_t));
  if (seg_flags) std::memcpy(seg_flags, hflags, nseg * sizeof(int));
  if (hoff[nseg] > capacity)
    return fail(c, VL_ERR_INVALID, "output capacity " + std::to_string(capacity) + " < " + std::to_string(hoff[nseg]) + " matches");
  if (!px_out || !X_out || !w_out) return fail(c, VL_ERR_INVALID, "null output array");
  prof_hook(c, kStageLift, true);
  c->launches += launch_lift_write(a, field_f64, mode, st);
  prof_hook(c, kStageLift, false);
  return check_launch(c);
}

extern "C" int vl_interp_depth(vl_ctx* c, const vl_lift_depth* depth, const double* pts, int64_t n, double* vals,
                               uint8_t* ok, void* stream) {
  if (!c || !depth || n < 0 || n > 0x7FFFFFFF) return fail(c, VL_ERR_INVALID, "bad argument");
  if (depth->width < 2 || depth->height < 2) return fail(c, VL_ERR_INVALID, "depth map must be at least 2x2");
  VL_CUDA(c, cudaSetDevice(c->device));
  LiftDepth D;
  std::memcpy(&D, depth, sizeof(D));
  c->launches += launch_interp(D, pts, (int)n, vals, ok, (cudaStream_t)stream);
  return check_launch(c);
}

extern "C" int vl_decode_depth(vl_ctx* c, const vl_lift_depth* depth, float* vals, uint8_t* valid, void* stream) {
  if (!c || !depth || !vals || !valid) return fail(c, VL_ERR_INVALID, "bad argument");
  VL_CUDA(c, cudaSetDevice(c->device));
  LiftDepth D;
  std::memcpy(&D, depth, sizeof(D));
  c->launches += launch_decode(D, (int64_t)D.w * D.h, vals, valid, (cudaStream_t)stream);
  return check_launch(c);
}

extern "C" int vl_robust_cost(vl_ctx* c, const double* q, const double* t, const double* px, const double* X,
                              const double* w, int64_t n, vl_intrinsics intr, int32_t loss, double scale,
                              double* cost_out, void* stream) {
  if (!c || !q || !t || !cost_out || n < 0 || n > 0x7FFFFFFF || (loss != 0 && loss != 1))
    return fail(c, VL_ERR_INVALID, "bad argument");
  if (!(scale > 0)) return fail(c, VL_ERR_INVALID, "scale must be positive");
  VL_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = ensure(c, c->scratch, 4096)) || (rc = ensure_host(c, 4096))) return rc;
  c->launches += launch_robust_cost(pose_from_host(q, t), px, X, w, (int)n,
                                    Intr{intr.fx, intr.fy, intr.cx, intr.cy}, loss, scale, (double*)c->scratch.p, st);
  if ((rc = check_launch(c))) return rc;
  double* h = (double*)c->h_pinned;
  VL_CUDA(c, cudaMemcpyAsync(h, c->scratch.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  VL_CUDA(c, cudaStreamSynchronize(st));
  *cost_out = h[0];
  return VL_OK;
}

extern "C" int vl_pose_residuals(vl_ctx* c, const double* q, const double* t, const double* px, const double* X,
                                 int64_t n, vl_intrinsics intr, double* res, double* z, double* J, void* stream) {
  if (!c || !q || !t || n < 0 || n > 0x7FFFFFFF) return fail(c, VL_ERR_INVALID, "bad argument");
  VL_CUDA(c, cudaSetDevice(c->device));
  c->launches += launch_residuals(pose_from_host(q, t), px, X, (int)n, Intr{intr.fx, intr.fy, intr.cx, intr.cy},
                                  res, z, J, (cudaStream_t)stream);
  return check_launch(c);
}

// ---- retrieval (retrieval.py:66-82) -----------------------------------------
namespace vl {
int launch_topk(const double* M, const int64_t* rank, int E, int D, const double* Qv, int Q, int K, int* out_idx,
                double* out_sim, int* bad, cudaStream_t st);
}

extern "C" int vl_retrieval_topk(vl_ctx* c, const double* db, const int64_t* id_rank, int32_t E, int32_t D,
                                 const double* queries, int32_t Q, int32_t k, int32_t* out_idx, double* out_sim,
                                 void* stream) {
  if (!c || E < 0 || D < 1 || Q < 0) return fail(c, VL_ERR_INVALID, "bad argument");
  if (k < 1) return fail(c, VL_ERR_INVALID, "k must be >= 1, got " + std::to_string(k));
  if (k > 32) return fail(c, VL_ERR_INVALID, "k must be <= 32 on the device path");
  if (Q == 0 || E == 0) return VL_OK;
  if (!db || !id_rank || !queries || !out_idx || !out_sim) return fail(c, VL_ERR_INVALID, "null array");
  VL_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = ensure(c, c->scratch, 4096)) || (rc = ensure_host(c, 4096))) return rc;
  int* dbad = (int*)c->scratch.p;
  VL_CUDA(c, cudaMemsetAsync(dbad, 0, sizeof(int), st));
  c->launches += launch_topk(db, id_rank, E, D, queries, Q, std::min(k, E), out_idx, out_sim, dbad, st);
  if ((rc = check_launch(c))) return rc;
  int* h = (int*)c->h_pinned;
  VL_CUDA(c, cudaMemcpyAsync(h, dbad, sizeof(int), cudaMemcpyDeviceToHost, st));
  VL_CUDA(c, cudaStreamSynchronize(st));
  if (*h) return fail(c, VL_ERR_INVALID, "query vector must be non-zero and finite");
  return VL_OK;
}

// ---- depth-map codecs (mapstore.py:96-134, :390-425) -------------------------
namespace vl {
struct CodecJob;
int launch_quantize(const CodecJob* jobs, int njobs, const uint32_t* thr, int nthr, int out16, int num_sms,
                    cudaStream_t st);
int launch_reduce_codes(const CodecJob* jobs, int njobs, int factor, int new_levels, int num_sms, cudaStream_t st);
}

static int check_codec_jobs(vl_ctx* c, const vl_depth_codec_job* jobs, int32_t njobs, bool codes_in) {
  if (njobs < 0 || (njobs > 0 && !jobs)) return fail(c, VL_ERR_INVALID, "bad argument");
  for (int j = 0; j < njobs; ++j) {
    const vl_depth_codec_job& J = jobs[j];
    const std::string tag = "map " + std::to_string(j) + ": ";
    if (J.width < 1 || J.height < 1 || (int64_t)J.width * J.height > INT32_MAX)
      return fail(c, VL_ERR_INVALID, tag + "bad shape");
    if (!J.values || !J.out || (!codes_in && !J.valid)) return fail(c, VL_ERR_INVALID, tag + "null array");
    if (codes_in ? (J.kind != 2 && J.kind != 3) : (J.kind != 0 && J.kind != 1))
      return fail(c, VL_ERR_INVALID, tag + "bad kind " + std::to_string(J.kind));
    if (codes_in && (J.levels < 1 || J.levels > 65535 || (J.kind == 2) != (J.levels <= 255)))
      return fail(c, VL_ERR_INVALID, tag + "levels out of range: " + std::to_string(J.levels));
  }
  return VL_OK;
}

extern "C" int vl_quantize_depth(vl_ctx* c, const vl_depth_codec_job* jobs, int32_t njobs, const float* thresholds,
                                 int32_t levels, void* stream) {
  if (!c) return VL_ERR_INVALID;
  if (levels < 1 || levels > 65535) return fail(c, VL_ERR_INVALID, "levels out of range: " + std::to_string(levels));
  if (levels > 1 && !thresholds) return fail(c, VL_ERR_INVALID, "null threshold table");
  int rc;
  if ((rc = check_codec_jobs(c, jobs, njobs, false))) return rc;
  if (njobs == 0) return VL_OK;
  VL_CUDA(c, cudaSetDevice(c->device));
  static_assert(sizeof(vl_depth_codec_job) == 40, "codec job layout");
  c->launches += launch_quantize((const CodecJob*)jobs, njobs, (const uint32_t*)thresholds, levels - 1,
                                 levels > 255, c->num_sms, (cudaStream_t)stream);
  return check_launch(c);
}

extern "C" int vl_reduce_depth_codes(vl_ctx* c, const vl_depth_codec_job* jobs, int32_t njobs, int32_t factor,
                                     int32_t new_levels, void* stream) {
  if (!c) return VL_ERR_INVALID;
  if (factor < 1) return fail(c, VL_ERR_INVALID, "resolution factors must be >= 1");
  if (new_levels < 1 || new_levels > 65535)
    return fail(c, VL_ERR_INVALID, "levels out of range: " + std::to_string(new_levels));
  int rc;
  if ((rc = check_codec_jobs(c, jobs, njobs, true))) return rc;
  if (njobs == 0) return VL_OK;
  VL_CUDA(c, cudaSetDevice(c->device));
  c->launches += launch_reduce_codes((const CodecJob*)jobs, njobs, factor, new_levels, c->num_sms,
                                     (cudaStream_t)stream);
  return check_launch(c);
}

// ---- dense depth triangulation (depthbuild.py:104-441) -----------------------
namespace vl {
struct TriMap;
struct TriView;
struct TriProblem;
struct TriObs;
struct TriConfig {
  double thr, conf_thr, refine_tol;
  int32_t min_inliers, max_refine_iters;
};
int launch_tri_maps(const TriMap* d_maps, int nmap, int max_pix, int max_views, const TriView* d_views, int f64,
                    const TriConfig& cfg, int num_sms, cudaStream_t st);
int launch_tri_rays(const TriProblem* d_probs, int nprob, int max_obs, const TriObs* d_obs, const TriConfig& cfg,
                    double* depth_out, int* count_out, double* hyp_out, int num_sms, cudaStream_t st);
}
static_assert(sizeof(vl_tri_config) == sizeof(vl::TriConfig) && sizeof(vl_tri_view) == 144 && sizeof(vl_tri_map) == 176 &&
                  sizeof(vl_tri_problem) == 56 && sizeof(vl_tri_obs) == 152, "tri layouts");

static int tri_config(vl_ctx* c, const vl_tri_config* cfg, TriConfig& out) {
  if (!cfg) return fail(c, VL_ERR_INVALID, "null config");
  if (!(cfg->angular_threshold_rad > 0)) return fail(c, VL_ERR_INVALID, "angular threshold must be positive");
  if (cfg->min_inliers < 1) return fail(c, VL_ERR_INVALID, "min_inliers must be >= 1");
  if (cfg->max_refine_iters < 0) return fail(c, VL_ERR_INVALID, "max_refine_iters must be >= 0");
  std::memcpy(&out, cfg, sizeof(out));
  return VL_OK;
}

extern "C" int vl_build_depth_maps(vl_ctx* c, const vl_tri_map* maps, int32_t nmap, const vl_tri_view* views,
                                   int32_t nviews, int32_t field_f64, const vl_tri_config* cfg, void* stream) {
  if (!c || nmap < 0 || nviews < 0 || (nmap && !maps) || (nviews && !views)) return fail(c, VL_ERR_INVALID, "bad argument");
  TriConfig tc;
  int rc;
  if ((rc = tri_config(c, cfg, tc))) return rc;
  if (nmap == 0) return VL_OK;
  int max_pix = 0, max_views = 1;
  for (int m = 0; m < nmap; ++m) {
    const vl_tri_map& M = maps[m];
    const std::string tag = "map " + std::to_string(m) + ": ";
    if (M.grid_w < 1 || M.grid_h < 1 || (int64_t)M.grid_w * M.grid_h > INT32_MAX) return fail(c, VL_ERR_INVALID, tag + "bad grid");
    if (M.nview < 1) return fail(c, VL_ERR_INVALID, tag + "need at least one correspondence field");
    if (M.nview > 128) return fail(c, VL_ERR_INVALID, tag + "at most 128 covisible views per map on the device path");
    if (M.view0 < 0 || (int64_t)M.view0 + M.nview > nviews) return fail(c, VL_ERR_INVALID, tag + "view range out of bounds");
    if (!M.depth || !M.valid) return fail(c, VL_ERR_INVALID, tag + "null output");
    max_pix = std::max(max_pix, M.grid_w * M.grid_h);
    max_views = std::max(max_views, M.nview);
  }
  for (int v = 0; v < nviews; ++v)
    if (!views[v].targets || !views[v].confidence) return fail(c, VL_ERR_INVALID, "view " + std::to_string(v) + ": null field");
  VL_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t mb = (size_t)nmap * sizeof(vl_tri_map), vb = (size_t)nviews * sizeof(vl_tri_view);
  if ((rc = ensure(c, c->tri_meta, mb + vb)) || (rc = ensure_host(c, mb + vb))) return rc;
  std::memcpy(c->h_pinned, maps, mb);
  std::memcpy((char*)c->h_pinned + mb, views, vb);
  VL_CUDA(c, cudaMemcpyAsync(c->tri_meta.p, c->h_pinned, mb + vb, cudaMemcpyHostToDevice, st));
  c->launches += launch_tri_maps((const TriMap*)c->tri_meta.p, nmap, max_pix, max_views,
                                 (const TriView*)((char*)c->tri_meta.p + mb), field_f64 ? 1 : 0, tc, c->num_sms, st);
  if ((rc = check_launch(c))) return rc;
  VL_CUDA(c, cudaStreamSynchronize(st));  // the pinned staging buffer is reused by the next call
  return VL_OK;
}

extern "C" int vl_triangulate_rays(vl_ctx* c, const vl_tri_problem* problems, int32_t nprob, const vl_tri_obs* obs,
                                   int32_t max_obs, const vl_tri_config* cfg, double* depth_out, int32_t* count_out,
                                   double* hyp_out, void* stream) {
  if (!c || nprob < 0 || (nprob && (!problems || !depth_out || !count_out))) return fail(c, VL_ERR_INVALID, "bad argument");
  if (max_obs < 0 || max_obs > 128) return fail(c, VL_ERR_INVALID, "at most 128 observations per problem on the device path");
  if (max_obs > 0 && !obs) return fail(c, VL_ERR_INVALID, "null observations");
  TriConfig tc;
  int rc;
  if ((rc = tri_config(c, cfg, tc))) return rc;
  if (nprob == 0) return VL_OK;
  VL_CUDA(c, cudaSetDevice(c->device));
  c->launches += launch_tri_rays((const TriProblem*)problems, nprob, std::max(max_obs, 1), (const TriObs*)obs, tc,
                                 depth_out, count_out, hyp_out, c->num_sms, (cudaStream_t)stream);
  return check_launch(c);
}
