// Batched, device-resident LO-RANSAC driver kernels (all but scoring).
//
// One "round" = one batch of `batch_size` minimal samples for every active
// query (posest.py:250-276):
//   k_sample   CTA/query : numpy-exact minimal sets (posest.py:252)
//   k_p3p_roots / k_p3p_polish : P3P solutions into per-sample slots (p3p.py:57)
//   k_compact  CTA/query : ordered hypothesis list + fp32 K[R|t] tiles,
//                          appends scoring work items
//   k_score    persistent grid (vl_score.cu): fp32 MSAC costs (posest.py:178)
//   k_scan     CTA/query : ordered first-better scan with LM local
//                          optimisation + adaptive stop (posest.py:257-276)
//              (its closing cluster also compacts the active-query list for
//              the next round: compact_active)
// After the last round k_final (CTA/query) classifies the full set and runs
// the Cauchy refinement (posest.py:284-299).
#include <algorithm>
#include <mutex>
#include <climits>
#include <cstddef>
#include <cstdlib>
#include "vl_internal.h"
#include "vl_lm.cuh"
#include "vl_p3p.cuh"

namespace vl {

// Initial phase-A prefix margin of exact scoring pruning: sA / NS = margin x
// best cost / typical hypothesis cost.  C3 step: 1.08 -> 53.3 ms, 1.05 ->
// 52.6, 1.03 -> 52.3, 1.00 -> 52.1, 0.97 -> 72.1 (most hypotheses survive the
// prefix and go to the tail); k_scan raises a query's margin by 10 % after a
// round in which more than a quarter of its hypotheses survived.
#ifndef VL_PRUNE_MARGIN
#define VL_PRUNE_MARGIN 1.03f
#endif

// ------------------------------------------------------------------ prep
// The per-query states come straight from the mapped pinned staging buffer
// (kernel loads over PCIe, not a copy-engine transfer, so a chunk never waits
// behind the host pipeline's bulk prefetch of the next chunk's matches).
// Block b admits query q0 + b at active-list position list_pos + b (staged
// admission appends a stage's queries behind the running ones).
__global__ void __launch_bounds__(256) k_prep(Work wk, Inputs in, const QState* __restrict__ host_qs, int q0,
                                              int list_pos) {
  const int q = q0 + blockIdx.x;
  QState& S = wk.qs[q];
  if (host_qs) {
    constexpr int kWords = sizeof(QState) / 4;
    static_assert(sizeof(QState) % 4 == 0, "QState word copy");
    const uint32_t* src = reinterpret_cast<const uint32_t*>(host_qs + q);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&S);
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x == 0) {
      wk.active_list[list_pos + blockIdx.x] = q;
      if (list_pos + blockIdx.x == 0) wk.item_count[0] = wk.item_count[1] = wk.item_count[2] = wk.item_count[3] = 0;
      if (blockIdx.x == 0) *wk.active_count = list_pos + (int)gridDim.x;  // admitted queries are active
    }
    __syncthreads();
  }
  const int64_t off = S.off, so = S.sub_off;
  const int stride = S.stride, nsub = S.nsub;
  const double cx = S.in.cx, cy = S.in.cy;
  int w_ok = 1;  // every fp32 weight >= 0 (scoring pruning: partial MSAC sums never decrease)
  for (int i = threadIdx.x; i < nsub; i += blockDim.x) {
    const int64_t src = off + (int64_t)i * stride;
    const double pu = in.px[2 * src], pv = in.px[2 * src + 1];
    const double X = in.X[3 * src], Y = in.X[3 * src + 1], Z = in.X[3 * src + 2];
    const double w = in.w[src];
    const int64_t d = so + i;
    wk.sub_pk[3 * d] = make_double2(X, Y);
    wk.sub_pk[3 * d + 1] = make_double2(Z, pu);
    wk.sub_pk[3 * d + 2] = make_double2(pv, w);
    // fp32 scoring record pair (SoA float2 of points 2k, 2k+1; sub_off is
    // even): X32, Y32, Z32, f32(cx - u), f32(cy - v), w32
    float* pr = reinterpret_cast<float*>(wk.sub32 + 3 * (d >> 1)) + (d & 1);
    pr[0] = (float)X;
    pr[2] = (float)Y;
    pr[4] = (float)Z;
    pr[6] = (float)(cx - pu);
    pr[8] = (float)(cy - pv);
    pr[10] = (float)w;
    w_ok &= (float)w >= 0.f ? 1 : 0;
    if ((nsub & 1) && i == nsub - 1)  // padding record: w = 0 adds +0
      for (int k = 0; k < 12; k += 2) pr[k + 1] = 0.f;
  }
  w_ok = __syncthreads_and(w_ok);
  if (threadIdx.x == 0) {
    if (wk.jump) pcg_jump_table(S.gen.inc, wk.jump + (int64_t)q * 2 * kJumpBits,
                                wk.jump + (int64_t)q * 2 * kJumpBits + kJumpBits);
    S.m_cache = ~0ull;
    S.spec_iters = S.iters;
    S.prune_ok = w_ok;
    S.sA = 0;
    S.cost_typ = 0.f;
    S.prune_m = VL_PRUNE_MARGIN;
  }
}

int launch_prep(const Work& wk, const Inputs& in, int q0, int nq, int list_pos, const QState* host_qs,
                cudaStream_t st) {
  if (nq <= 0) return 0;
  k_prep<<<nq, 256, 0, st>>>(wk, in, host_qs, q0, list_pos);
  return 1;
}

// ------------------------------------------------------------------ sampling
// Speculative parallel generation: sample i assumes no Lemire rejection
// happened in samples [i0, i); the first sample that would reject is redone
// exactly by one thread and speculation restarts after it.
// Speculation rounds start from a base state computed once by thread 0 (one
// O(log n) pcg_advance); each thread then jumps only its own offset within
// the batch through the block's 2^k jump table (a few affine compositions
// instead of a full O(log n) advance per thread).
// With a per-query jump table `tab` (k_prep) and the cached base of the
// previous round (`cache_st` advanced `*cache_m` steps), the base of the
// first window is a short table jump (one batch of draws ahead) instead of an
// O(log n) advance from the seed state; both give the same state.
template <int NT>
__device__ void sample_batch(const GenState& g, uint64_t& pos, int64_t n, int bn, int* out,
                             const u128* tab = nullptr, u128* cache_st = nullptr, uint64_t* cache_m = nullptr) {
  __shared__ int s_first;
  __shared__ unsigned long long s_pos;
  __shared__ u128 s_tmul[kJumpBits], s_tplus[kJumpBits], s_base;
  __shared__ unsigned long long s_m0;
  const int D = draws_per_sample(n);
  if (tab) {
    if (threadIdx.x < kJumpBits) {
      s_tmul[threadIdx.x] = tab[threadIdx.x];
      s_tplus[threadIdx.x] = tab[kJumpBits + threadIdx.x];
    }
    __syncthreads();
  } else if (threadIdx.x == 0) {
    pcg_jump_table(g.inc, s_tmul, s_tplus);
  }
  int i0 = 0;
  while (i0 < bn) {
    if (threadIdx.x == 0) {
      s_first = INT_MAX;
      const uint64_t q0 = pos >= (uint64_t)g.has0 ? pos - g.has0 : 0;  // first non-buffered word
      s_m0 = q0 >> 1;
      const uint64_t want = s_m0 + 1, have = cache_m ? *cache_m : ~0ull;
      if (have != ~0ull && want >= have && want - have < (1ull << kJumpBits))
        s_base = pcg_advance_tab(*cache_st, want - have, s_tmul, s_tplus);
      else
        s_base = pcg_advance(g.state, g.inc, want);
    }
    __syncthreads();
    // the speculative window spans at most NT samples at a time: offsets < 2^kJumpBits words
    for (int i = i0 + threadIdx.x; i < bn; i += NT) {
      WordReader rd;
      const uint64_t off = (uint64_t)D * (uint64_t)(i - i0);
      if (off < (1ull << (kJumpBits - 1)))
        reader_init_from(rd, g, pos + off, s_base, s_m0, s_tmul, s_tplus);
      else
        rd.init(g, pos + off);
      int64_t v[3];
      if (choice3(rd, (uint32_t)n, false, v, nullptr)) {
        out[3 * i] = (int)v[0];
        out[3 * i + 1] = (int)v[1];
        out[3 * i + 2] = (int)v[2];
      } else {
        atomicMin(&s_first, i);
      }
    }
    __syncthreads();
    const int r = s_first;
    if (r == INT_MAX) {
      pos += (uint64_t)D * (uint64_t)(bn - i0);
      break;
    }
    if (threadIdx.x == 0) {
      const uint64_t p = pos + (uint64_t)D * (uint64_t)(r - i0);
      WordReader rd;
      rd.init(g, p);
      int64_t v[3];
      int used = 0;
      choice3(rd, (uint32_t)n, true, v, &used);
      out[3 * r] = (int)v[0];
      out[3 * r + 1] = (int)v[1];
      out[3 * r + 2] = (int)v[2];
      s_pos = p + (uint64_t)used;
    }
    __syncthreads();
    pos = s_pos;
    i0 = r + 1;
    __syncthreads();
  }
  if (cache_m && threadIdx.x == 0) {  // the last window's base
    *cache_st = s_base;
    *cache_m = s_m0 + 1;
  }
}

// NT threads per query: 256 for big batches, 1024 when few queries are active
// (single-query latency: one speculative draw per thread)
// Per-query kernels return for list positions >= *active_count: the host may
// queue a round with a stale (larger) grid before it has read the previous
// round's count (one-round lookahead, vl_ransac_pnp).
template <int NT>
__global__ void __launch_bounds__(NT) k_sample(Work wk, RansacParams p) {
  pdl_enter();
  if ((int)blockIdx.x >= *wk.active_count) return;
  const int q = wk.active_list[blockIdx.x];
  QState& S = wk.qs[q];
  const int64_t rem = p.max_iterations - S.spec_iters;
  const int bn = (int)(rem < p.batch_size ? rem : p.batch_size);
  uint64_t pos = S.rng_pos;
  sample_batch<NT>(S.gen, pos, S.n, bn, wk.samples + (int64_t)q * wk.B * 3,
                   wk.jump ? wk.jump + (int64_t)q * 2 * kJumpBits : nullptr, &S.st_cache, &S.m_cache);
  if (threadIdx.x == 0) {
    S.rng_pos = pos;
    S.bn_p[wk.par] = bn;
    S.spec_iters += bn;
    S.iters_p[wk.par] = S.spec_iters;
  }
}

__global__ void __launch_bounds__(256) k_sample_one(GenState g, uint64_t pos0, int64_t n, int count,
                                                    int* out, uint64_t* pos_out) {
  uint64_t pos = pos0;
  sample_batch<256>(g, pos, n, count, out);
  if (threadIdx.x == 0) *pos_out = pos;
}

int launch_sample(const GenState& g, uint64_t pos0, int64_t n, int count, int* out, uint64_t* pos_out,
                  cudaStream_t st) {
  k_sample_one<<<1, 256, 0, st>>>(g, pos0, n, count, out, pos_out);
  return 1;
}

// ------------------------------------------------------------------ P3P
__device__ __forceinline__ void bearing(const double* px, const Intr& in, double* f) {
  const double b0 = (px[0] - in.cx) / in.fx, b1 = (px[1] - in.cy) / in.fy;
  const double nr = sqrt(dadd(dadd(dmul(b0, b0), dmul(b1, b1)), 1.0));
  f[0] = b0 / nr;
  f[1] = b1 / nr;
  f[2] = 1.0 / nr;
}

// P3P in two kernels (one kernel with both phases thrashed the instruction
// cache: ncu stall_no_inst 34 %, and its register / smem footprint capped
// occupancy at 12 warps per SM).
//  k_p3p_roots  lane = minimal sample: gate, resultant quartic, real positive
//               roots, distance-triple candidates (p3p.py:91-231); the
//               sample's geometry and candidates go to global scratch.
//  k_p3p_polish warp = 32 consecutive samples: their candidates are compacted
//               in (sample, root) order into shared memory and polished 32 at a
//               time (lane = candidate: Newton + Procrustes + contract), so the
//               ~1.5 candidates per sample keep every lane busy; each sample's
//               owner lane then dedups its candidates in order into the
//               sample's solution slots (<= 4) — the reference's order.
// The arithmetic is the single-kernel version's, function for function.
static_assert(sizeof(P3PGeo) == kGeoDoubles * sizeof(double) && kMaxCand == kMaxCandSlots, "P3P scratch layout");
constexpr int kP3PRootThreads = 128;
constexpr int kP3PThreads = 64;
struct CandRec {
  double s0, s1, s2;
  int lane, pad;
};

// fp32 scoring row of one hypothesis: diag(fx, fy, 1) [R | t] (R row-major,
// t in sl[9..11]), folded in fp64 and rounded once, stored SoA with column
// stride cs (k_score reads entry c of hypothesis h at P[c * cs + h]).
__device__ __forceinline__ void store_p32(float* P, int64_t cs, double fx, double fy, const double* sl, int es = 1) {
  P[0 * cs] = (float)(fx * sl[0 * es]);
  P[1 * cs] = (float)(fx * sl[1 * es]);
  P[2 * cs] = (float)(fx * sl[2 * es]);
  P[3 * cs] = (float)(fx * sl[9 * es]);
  P[4 * cs] = (float)(fy * sl[3 * es]);
  P[5 * cs] = (float)(fy * sl[4 * es]);
  P[6 * cs] = (float)(fy * sl[5 * es]);
  P[7 * cs] = (float)(fy * sl[10 * es]);
  P[8 * cs] = (float)sl[6 * es];
  P[9 * cs] = (float)sl[7 * es];
  P[10 * cs] = (float)sl[8 * es];
  P[11 * cs] = (float)sl[11 * es];
}

#ifndef VL_P3P_ROOT_MINB
#define VL_P3P_ROOT_MINB 5  // measured: 5 resident CTAs (96 regs) beat 4 (112 regs)
#endif
#ifndef VL_P3P_POLISH_MINB
#define VL_P3P_POLISH_MINB 8  // measured: 128-register cap, 8 CTAs
#endif
__global__ void __launch_bounds__(kP3PRootThreads, VL_P3P_ROOT_MINB) k_p3p_roots(Work wk, Inputs in) {
  pdl_enter();
  if ((int)blockIdx.x >= *wk.active_count) return;
  const int q = wk.active_list[blockIdx.x];
  const QState& S = wk.qs[q];
  const int s = blockIdx.y * kP3PRootThreads + threadIdx.x;
  if (s >= S.bn_p[wk.par]) return;
  const int64_t si = (int64_t)q * wk.B + s;
  const int* smp = wk.samples + si * 3;
  double f[9], P[9];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int64_t r = S.off + smp[k];
    bearing(in.px + 2 * r, S.in, f + 3 * k);
    P[3 * k] = in.X[3 * r];
    P[3 * k + 1] = in.X[3 * r + 1];
    P[3 * k + 2] = in.X[3 * r + 2];
  }
  P3PGeo g;
  double quart[5], vs[4];
  int nc = 0;
  const int64_t grp = (int64_t)q * ((wk.B + 31) / 32) + s / 32;  // warp-blocked SoA scratch
  const int ln = s & 31;
  if (p3p_setup(f, P, g, quart)) {
    const int nv = quartic_real_pos_roots(quart, vs);
    if (nv) nc = p3p_candidates(g, vs, nv, wk.p3p_cand + grp * (3 * kMaxCand * 32) + ln, 3 * 32, 32);
  }
  if (nc) {
    const double* gd = reinterpret_cast<const double*>(&g);
    double* dst = wk.p3p_geo + grp * (kGeoDoubles * 32) + ln;
#pragma unroll
    for (int k = 0; k < kGeoDoubles; ++k) dst[32 * k] = gd[k];
  }
  wk.p3p_nc[si] = nc;
}

__global__ void __launch_bounds__(kP3PThreads, VL_P3P_POLISH_MINB) k_p3p_polish(Work wk) {
  pdl_enter();
  __shared__ CandRec cand[kP3PThreads / 32][32 * kMaxCand];
  __shared__ double res[kP3PThreads / 32][32][13];
  if ((int)blockIdx.x >= *wk.active_count) return;
  const int q = wk.active_list[blockIdx.x];
  const QState& S = wk.qs[q];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int s = blockIdx.y * kP3PThreads + threadIdx.x;
  const int64_t si = (int64_t)q * wk.B + s;
  const bool live = s < S.bn_p[wk.par];
  const int nc = live ? wk.p3p_nc[si] : 0;
  // warp exclusive scan of candidate counts
  int incl = nc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int base = incl - nc;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  // this warp's 32 samples are one block of the SoA scratch (s is a multiple of 32 at lane 0)
  const int64_t grp = (int64_t)q * ((wk.B + 31) / 32) + s / 32;
  const double* cs = wk.p3p_cand + grp * (3 * kMaxCand * 32) + lane;
  for (int i = 0; i < nc; ++i)
    cand[wid][base + i] = CandRec{cs[32 * (3 * i)], cs[32 * (3 * i + 1)], cs[32 * (3 * i + 2)], lane, 0};
  __syncwarp();
  double* slot = slot_ptr(wk, q, s, 0);  // element e of kept solution k: slot[32 * (12 k + e)]
  const double* geo = wk.p3p_geo + grp * (kGeoDoubles * 32);
  const double ttol = nc ? kDedupTol * sqrt(geo[32 * (offsetof(P3PGeo, scale2) / 8) + lane]) : 0.0;
  int kept = 0;
  for (int ch = 0; ch < total; ch += 32) {
    const int j = ch + lane;
    if (j < total) {
      const CandRec cr = cand[wid][j];
      P3PGeo g;
      {
        double* gd = reinterpret_cast<double*>(&g);
#pragma unroll
        for (int k = 0; k < kGeoDoubles; ++k) gd[k] = geo[32 * k + cr.lane];
      }
      double R[9], t[3];
      const double sv[3] = {cr.s0, cr.s1, cr.s2};
      const bool ok = p3p_polish(g, sv, R, t);
#pragma unroll
      for (int i = 0; i < 9; ++i) res[wid][lane][i] = R[i];
#pragma unroll
      for (int i = 0; i < 3; ++i) res[wid][lane][9 + i] = t[i];
      res[wid][lane][12] = ok ? 1.0 : 0.0;
    }
    __syncwarp();
    const int e0 = max(base, ch), e1 = min(base + nc, ch + 32);
    for (int e = e0; e < e1; ++e) {
      const double* rr = res[wid][e - ch];
      if (rr[12] == 0.0 || kept >= kMaxSolPerSample) continue;
      bool dup = false;
      for (int k = 0; k < kept && !dup; ++k) {
        double sk[12];
#pragma unroll
        for (int i = 0; i < 12; ++i) sk[i] = slot[32 * (12 * k + i)];
        dup = p3p_is_dup(rr, rr + 9, sk, sk + 9, ttol);
      }
      if (dup) continue;
      for (int i = 0; i < 12; ++i) slot[32 * (12 * kept + i)] = rr[i];
      // the fp32 scoring row, at slot column kept * B + s of the query
      store_p32(wk.P32s + (int64_t)q * 12 * wk.HCAP + (int64_t)kept * wk.B + s, wk.HCAP, S.in.fx, S.in.fy, rr);
      ++kept;
    }
    __syncwarp();
  }
  if (live) wk.slot_cnt[si] = kept;
}

__global__ void __launch_bounds__(128) k_p3p_batch(const double* f, const double* P, int B, double* slots,
                                                   int* cnt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= B) return;
  double Rs[36], ts[12];
  const int c = p3p_solve_one(f + 9 * s, P + 9 * s, Rs, ts);
  double* slot = slots + (int64_t)s * 48;
  for (int k = 0; k < c; ++k) {
    for (int i = 0; i < 9; ++i) slot[12 * k + i] = Rs[9 * k + i];
    for (int i = 0; i < 3; ++i) slot[12 * k + 9 + i] = ts[3 * k + i];
  }
  cnt[s] = c;
}

// ------------------------------------------------------------------ compaction
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  int base = 0, tot = 0;
  for (int w = 0; w < NT / 32; ++w) {
    const int t = warp_tot[w];
    if (w < wid) base += t;
    tot += t;
  }
  __syncthreads();
  total = tot;
  return base + x - v;
}

// ordered gather of the per-sample solution slots (standalone p3p_solve_batch)
__global__ void __launch_bounds__(1024) k_p3p_gather(const double* slots, const int* cnt, int B, double* R_out,
                                                    double* t_out, int64_t* idx_out, int* m_out) {
  __shared__ int warp_tot[32];
  int running = 0;
  for (int base = 0; base < B; base += 1024) {
    const int s = base + threadIdx.x;
    const int c = s < B ? cnt[s] : 0;
    int total;
    const int ex = block_excl_scan<1024>(c, warp_tot, total);
    for (int k = 0; k < c; ++k) {
      const int m = running + ex + k;
      const double* sl = slots + (int64_t)s * 48 + 12 * k;
      for (int i = 0; i < 9; ++i) R_out[9 * (int64_t)m + i] = sl[i];
      for (int i = 0; i < 3; ++i) t_out[3 * (int64_t)m + i] = sl[9 + i];
      idx_out[m] = s;
    }
    running += total;
  }
  if (threadIdx.x == 0) *m_out = running;
}

int launch_p3p_batch(const double* f, const double* P, int B, double* slots, int* cnt, double* R_out,
                     double* t_out, int64_t* idx_out, int* m_out, cudaStream_t st) {
  if (B <= 0) return 0;
  k_p3p_batch<<<(B + 127) / 128, 128, 0, st>>>(f, P, B, slots, cnt);
  k_p3p_gather<<<1, 1024, 0, st>>>(slots, cnt, B, R_out, t_out, idx_out, m_out);
  return 2;
}

// Standalone scoring (vl_score_hypotheses): rows of caller-given hypotheses
// for query 0 of a one-query workspace, plus that round's score items.
__global__ void k_hyp_rows(Work wk, const double* R, const double* t, int H, int fine) {
  const QState& S = wk.qs[0];
  for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    double sl[12];
    for (int i = 0; i < 9; ++i) sl[i] = R[9 * (int64_t)h + i];
    for (int i = 0; i < 3; ++i) sl[9 + i] = t[3 * (int64_t)h + i];
    store_p32(wk.P32 + h, wk.HCAP, S.in.fx, S.in.fy, sl);
  }
  const int tile_h = fine ? kScoreTileHypsFine : kScoreTileHyps;
  const int spi = fine ? 1 : kScoreItemSplits;
  const int ntile = (H + tile_h - 1) / tile_h, ngroups = (S.nsplit + spi - 1) / spi;
  const int nitems = ntile * ngroups;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nitems; i += gridDim.x * blockDim.x) {
    ScoreItem it;
    it.q = 0;
    it.tile = i / ngroups;
    it.split = (i % ngroups) * spi;
    it.nsplit = min(spi, S.nsplit - it.split);
    wk.items[i] = it;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < wk.TCAP; i += gridDim.x * blockDim.x) wk.tile_cnt[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    wk.item_count[0] = nitems;
    wk.item_count[1] = 0;
  }
}

int launch_hyp_rows(const Work& wk, const double* R, const double* t, int H, int fine, cudaStream_t st) {
  k_hyp_rows<<<std::max(1, std::min(148, (H + 255) / 256)), 256, 0, st>>>(wk, R, t, H, fine);
  return 1;
}

// mode 0 (full round): order the hypotheses, items for all of them.  Split
// rounds: mode 1 (head) orders them and emits items only for the first
// kHeadHyps of queries without a best pose; mode 2 (rest) emits the items of
// the remaining hypotheses (all of them for queries that had a best pose),
// pruned against the best the head scan found.
// head size (A/B, ms per step C3a / C3 pruned / C5): 192: 11.10 / 48.74 /
// 6.93, 256: 11.68 / 49.28 / 7.14, 384: 11.29 / 48.74 / 7.12, 576: 12.65 /
// 50.23 / 7.41.  (P(no all-inlier sample among the head's ~128 samples) at
// 30 % inliers: 3 %; a weak head best only weakens the pruning, never the result)
#ifndef VL_HEAD_HYPS
#define VL_HEAD_HYPS 192
#endif
constexpr int kHeadHyps = VL_HEAD_HYPS;

template <int NT>
__global__ void __launch_bounds__(NT) k_compact(Work wk, int fine, int mode) {
  pdl_enter();
  __shared__ int warp_tot[32];
  __shared__ int s_item0;
  if ((int)blockIdx.x >= *wk.active_count) return;
  const int q = wk.active_list[blockIdx.x];
  QState& S = wk.qs[q];
  int nh;
  if (mode != 2) {
    const int bn = S.bn_p[wk.par];
    int running = 0;
    for (int base = 0; base < bn; base += NT) {
      const int s = base + threadIdx.x;
      const int c = s < bn ? wk.slot_cnt[(int64_t)q * wk.B + s] : 0;
      int total;
      const int ex = block_excl_scan<NT>(c, warp_tot, total);
      // hypothesis h -> its solution slot k * B + s
      for (int k = 0; k < c; ++k) wk.hsrc[(int64_t)q * wk.HCAP + running + ex + k] = k * wk.B + s;
      running += total;
    }
    nh = running;
#if VL_P32_COPY
    __syncthreads();
    // the fp32 rows (written by k_p3p_polish at the slot columns) in
    // hypothesis order: the scorer then reads them with no indirection
    const int* hq = wk.hsrc + (int64_t)q * wk.HCAP;
    const float* src = wk.P32s + (int64_t)q * 12 * wk.HCAP;
    float* dst = wk.P32 + (int64_t)q * 12 * wk.HCAP;
    for (int h = threadIdx.x; h < nh; h += NT) {
      const int col = hq[h];
#pragma unroll
      for (int e = 0; e < 12; ++e) dst[(int64_t)e * wk.HCAP + h] = src[(int64_t)e * wk.HCAP + col];
    }
#endif
  } else {
    nh = S.nh;
  }
  int lo = 0, hi = nh;
  if (mode == 1) hi = S.has_best ? 0 : min(nh, kHeadHyps);
  else if (mode == 2) lo = S.h_hi;
  // score work items: coarse (768-hypothesis tiles x 4 splits) for big batches,
  // fine (256 x 1) when the batch is too small to fill the GPU otherwise;
  // tiles count from h_lo
  // (fine == 2, "medium": a single query's round, 256-hypothesis tiles x 4-split items)
  const int tile_h = fine ? kScoreTileHypsFine : kScoreTileHyps;
  const int spi = fine == 1 ? 1 : kScoreItemSplits;
  const int ntile = (hi - lo + tile_h - 1) / tile_h;
  // exact pruning (coarse rounds, a best pose known, non-negative weights):
  // score the first sA splits of every hypothesis, where sA / NS is the best
  // cost over the typical hypothesis cost of the last fully scored round
  // (plus 8 %): a typical hypothesis' prefix then already exceeds the best
  // cost, and only the others are finished (k_score_tail).  The last phase-A
  // item of a tile may cover only the first sA mod 4 splits of its group.
  int sA = S.nsplit;
  if (mode != 1 && wk.prune && !fine && S.prune_ok && S.has_best && S.cost_typ > 0.f) {
    const double f = S.best_cost / (double)S.cost_typ * (double)S.prune_m;
    if (f < 1.0) sA = max(1, min(S.nsplit, (int)ceil(f * S.nsplit)));
  }
  const int ngroups = (sA + spi - 1) / spi;
  // hypothesis-split mode: tile (q, t) belongs to rank (q*TCAP + t) mod size;
  // the other ranks leave its costs at zero for the SUM all-reduce
  const int size = wk.split_size;
  const int t0 = size > 1 ? (int)((((int64_t)wk.split_rank - (int64_t)q * wk.TCAP) % size + size) % size) : 0;
  const int nown = t0 < ntile ? (ntile - 1 - t0) / size + 1 : 0;
  const int nitems = nown * ngroups;
  for (int t = threadIdx.x; t < ntile; t += NT) wk.tile_cnt[(int64_t)q * wk.TCAP + t] = 0;
  if (size > 1)
    for (int h = threadIdx.x; h < nh; h += NT)
      if ((h / tile_h) % size != t0) wk.cost32[(int64_t)q * wk.HCAP + h] = 0.f;
  if (threadIdx.x == 0) {
    if (mode != 2) {
      S.nh = nh;
      S.hyps += nh;
      S.evals += (int64_t)nh * S.nsub;
    }
    S.h_lo = lo;
    S.h_hi = hi;
    S.sA = sA;
    S.nsurv = 0;
    S.tiles_closed = 0;
    s_item0 = nitems > 0 ? atomicAdd(wk.item_count, nitems) : 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nitems; i += NT) {
    ScoreItem it;
    it.q = q;
    it.tile = t0 + (i / ngroups) * size;
    it.split = (i % ngroups) * spi;
    it.nsplit = min(spi, sA - it.split);
    const int64_t pos = (int64_t)s_item0 + i;
    if (pos < wk.item_cap) wk.items[pos] = it;
  }
}

// ------------------------------------------------------------------ scan + LO + stop
__device__ __forceinline__ int64_t required_iters_dev(double eps, double eta, int64_t cap) {
  eps = fmin(fmax(eps, 0.0), 1.0);
  if (eps <= 0.0) return cap;
  if (eps >= 1.0) return 1;
  const double den = log1p(-pow(eps, 3.0));
  if (den == 0.0) return cap;
  const double nn = ceil(log(eta) / den);
  double v = fmax(nn, 1.0);
  if (v > (double)cap) return cap;
  return (int64_t)v;
}

#ifndef VL_LO_NT
#define VL_LO_NT 256   // threads of the per-query LO kernels (k_scan, k_final)
#endif
#ifndef VL_LO_MINB
#define VL_LO_MINB 2   // resident CTAs per SM (bounds the LO working set held in L2)
#endif
constexpr int kScanThreads = VL_LO_NT;

// Active-list compaction after a round (the loop condition of posest.py:250):
// queries still active keep their order.  Run by one CTA once every query's
// scan has finished (the closing cluster of k_scan, after an atomic ticket);
// the other CTAs' QState writes are read through L2.
template <int NT>
__device__ void compact_active(Work wk, int nactive) {
  __shared__ int warp_tot[32];
  int running = 0;
  for (int base = 0; base < nactive; base += NT) {
    const int i = base + threadIdx.x;
    const int q = i < nactive ? __ldcg(wk.active_list + i) : -1;
    const int a = (q >= 0 && __ldcg(&wk.qs[q].active)) ? 1 : 0;
    int total;
    const int ex = block_excl_scan<NT>(a, warp_tot, total);
    // (in place when next_list == active_list: write index <= read index)
    if (a) wk.next_list[running + ex] = q;
    running += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *wk.next_count = running;
    if (wk.host_count) *(volatile int*)wk.host_count = running;  // mapped pinned: read after the stream sync
    wk.item_count[0] = 0;  // items appended next round
    wk.item_count[1] = 0;  // scoring work cursor
    wk.item_count[2] = 0;  // k_scan completion ticket
    wk.item_count[3] = 0;  // scoring tail tasks
  }
}

// costs_smem: the round's fp32 costs are copied to shared memory (HCAP floats
// after the staging ring) unless a huge batch_size would not fit, in which
// case the scan reads them from L2.
// mode (k_compact's): 0 full round, 1 head of a split round (hypotheses
// [h_lo, h_hi) only; no stop rule, the active list stays), 2 rest of it.
__global__ void __launch_bounds__(kScanThreads, VL_LO_MINB) k_scan(Work wk, RansacParams p, int costs_smem,
                                                                  int mode, int fine) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  double2* ring = reinterpret_cast<double2*>(dyn_smem);  // kStageBytes (TMA staging ring)
  __shared__ uint64_t stage_bar[kStageN];
  __shared__ LMShared<kScanThreads> sm;
  __shared__ Pose s_start;
  __shared__ int s_last;
  // the active count of this round (the grid may be a stale superset, see
  // vl_ransac_pnp's lookahead); read once: the closing cluster rewrites it
  const int nact = *wk.active_count;
  const int nlist = min((int)(gridDim.x / cl_size()), nact);
  if ((int)(blockIdx.x / cl_size()) >= nlist) return;  // whole cluster
  const int q = wk.active_list[blockIdx.x / cl_size()];
  QState& S = wk.qs[q];
  const int hlo = S.h_lo, nh = S.h_hi;  // this phase's hypotheses [hlo, nh)
  // final fp32 costs (canonical order, reduced by the scorer's tile tickets)
  const float* cq = wk.cost32 + (int64_t)q * wk.HCAP;
  const float* costs = cq;
  if (costs_smem) {
    float* cs = reinterpret_cast<float*>(dyn_smem + kStageBytes);  // [HCAP]
    for (int h = hlo + threadIdx.x; h < nh; h += kScanThreads) cs[h] = __ldcg(cq + h);
    costs = cs;
  }
  __syncthreads();
  // typical hypothesis cost (mean fp32 cost) of fully scored hypotheses: sizes
  // the next pruning prefix (k_compact); pruned phases keep it
  float cost_typ = S.cost_typ, prune_m = S.prune_m;
  if (S.sA < S.nsplit && S.nsurv * 4 > nh - hlo) prune_m *= 1.1f;  // pruned, many survivors
  if (wk.prune && !fine && nh > hlo && S.sA >= S.nsplit) {  // (fine rounds never prune)
    double acc[1] = {0.0};
    for (int h = hlo + threadIdx.x; h < nh; h += kScanThreads) acc[0] += (double)costs[h];
    block_sum<kScanThreads, 1>(acc, sm.scratch, sm.red);
    const double m = sm.red[0] / (nh - hlo);
    cost_typ = m < 3.0e38 ? (float)m : 0.f;
    __syncthreads();
  }
  const Intr in = S.in;
  const StagedPts sub{wk.sub_pk + 3 * S.sub_off, S.nsub, ring, stage_bar};
  double best_cost = S.best_cost;
  int has_best = S.has_best;
  Pose best = S.best;
  int64_t lo_calls = 0;
  int64_t best_cnt = S.best_cnt_valid ? S.best_sub_cnt : -1;  // -1: not known for `best`
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int h0 = hlo;
  while (h0 < nh) {
    // the first h >= h0 with cost < best: every thread stops at its own first
    // hit (strided), one block minimum (a round without an LO: one reduction
    // instead of one per 256 hypotheses)
    int f = INT_MAX;
    for (int i = h0 + threadIdx.x; i < nh; i += kScanThreads)
      if ((double)costs[i] < best_cost) {
        f = i;
        break;
      }
    f = (int)__reduce_min_sync(0xffffffffu, (unsigned)f);
    if (lane == 0) sm.ibuf[wid] = f;
    __syncthreads();
    int found = INT_MAX;
    for (int w = 0; w < kScanThreads / 32; ++w) found = min(found, sm.ibuf[w]);
    __syncthreads();
    if (found == INT_MAX) break;
    best_cost = (double)costs[found];
    has_best = 1;
    if (threadIdx.x == 0) {
      const int src = wk.hsrc[(int64_t)q * wk.HCAP + found];  // k * B + s
      const double* sp = slot_ptr(wk, q, src % wk.B, src / wk.B);
      double sl[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) sl[i] = sp[32 * i];
      pose_from_Rt(sl, sl + 9, s_start);
    }
    __syncthreads();
    const Pose start = s_start;
    lm_refine<kScanThreads>(sm, sub, in, start, kTruncated, p.tau, p.lm_max_iters, 1e-10, 1e-12, nullptr,
                            nullptr);
    const Pose lo = sm.cur;
    set_eval_pose(sm, lo);
    msac_pass<kScanThreads>(sm, sub, in, p.tau, nullptr);
    const double lo_cost = sm.red[0];
    if (lo_cost < best_cost) {
      best_cost = lo_cost;
      best = lo;
      best_cnt = (int64_t)sm.red[1];  // this pass is the stop rule's msac_score of the new best
    } else {
      best = start;
      best_cnt = -1;
    }
    ++lo_calls;
    h0 = found + 1;
    __syncthreads();
  }
  int active = 1;
  const int64_t iters_r = S.iters_p[wk.par];  // samples drawn up to this round
  if (mode != 1 && has_best) {
    // the stop rule's subset inlier count (posest.py:269-273): computed once
    // per best pose — an unchanged best (most rounds after the first) or a
    // best just set by an accepted LO (its msac pass above) reuses the count,
    // which is the same pass over the same pose and subset, hence identical
    if (best_cnt < 0) {
      set_eval_pose(sm, best);
      msac_pass<kScanThreads>(sm, sub, in, p.tau, nullptr);
      best_cnt = (int64_t)sm.red[1];
    }
    const int64_t need = required_iters_dev((double)best_cnt / (double)S.nsub, p.eta, p.max_iterations);
    if (iters_r >= need) active = 0;
  }
  if (iters_r >= p.max_iterations) active = 0;
  __syncthreads();
  if (cl_size() > 1) cl_sync();  // every CTA of the cluster has read S
  if (threadIdx.x == 0 && cl_rank() == 0) {
    S.best_cost = best_cost;
    S.has_best = has_best;
    S.best = best;
    S.lo_calls += lo_calls;
    if (mode != 1) {  // (head phase: the round goes on)
      S.active = active;
      S.iters = iters_r;  // the round is scanned: its samples count
      S.rounds += 1;
    }
    S.best_sub_cnt = best_cnt;
    S.best_cnt_valid = best_cnt >= 0 ? 1 : 0;
    S.cost_typ = cost_typ;
    S.prune_m = prune_m;
  }
  // the last cluster to finish compacts the active list for the next round
  // (was a separate one-CTA kernel per round: ~8.6 us of launch + drain per
  // round on single-query configs)
  if (cl_rank() == 0) {
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(wk.item_count + 2, 1) == nlist - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      if (mode != 1) {
        compact_active<kScanThreads>(wk, nlist);
      } else if (threadIdx.x == 0) {  // head phase: only the work counters restart
        wk.item_count[0] = wk.item_count[1] = wk.item_count[2] = wk.item_count[3] = 0;
      }
    }
  }
}




// Cluster size for a per-query kernel: spread few queries over up to 8 SMs
// each (single-query latency), keep one CTA per query when the batch alone
// fills the GPU (`slots` = resident CTAs the GPU holds).
static int pick_cluster(int nq, int slots) {
  int cs = 1;
  while (cs < 8 && (int64_t)nq * cs * 2 <= slots) cs *= 2;
  return cs;
}

template <typename... KArgs, typename... Args>
static void launch_clustered(void (*k)(KArgs...), int nq, int block, size_t smem, int cs, cudaStream_t st,
                             bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nq * cs, 1, 1);
  cfg.blockDim = dim3(block, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}

// A plain launch, optionally as a programmatic dependent launch (see pdl_enter).
template <typename... KArgs, typename... Args>
static void launch_k(void (*k)(KArgs...), dim3 grid, int block, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, args...);
}

// PDL for every round launch (VISLOC_PDL=0 turns it off): C1 1.25 -> 1.10 ms,
// C4 10.9 -> 9.8 ms, C2 1.71 -> 1.60 ms; big batches +0.05-0.4 %
static bool use_pdl(int) {
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("VISLOC_PDL");
    mode = e ? atoi(e) : 1;
  }
  return mode != 0;
}

// coarse scoring items unless the whole batch would not fill ~3 waves of SMs
bool round_is_fine(const Work& wk, int nactive, int num_sms) {
  const int coarse_items = nactive * 2 * ((wk.NSPLIT + kScoreItemSplits - 1) / kScoreItemSplits);
  return coarse_items < 3 * num_sms;
}

// ---------------------------------------------------------- hypothesis-split argmin
// BASELINE's packed (score, index) variant of the hypothesis split (SURVEY
// §8e): per active query, the minimum over this rank's OWN hypotheses of
// key = float_bits(cost) << 32 | h (costs are >= 0, so the bit pattern orders
// like the value and ties go to the lowest index); other queries keep
// INT64_MAX.  A MIN all-reduce of the keys (8 B per query) then selects the
// batch's best hypothesis on every rank.
__global__ void __launch_bounds__(256) k_split_argmin(Work wk, int tile_h, long long* keys) {
  __shared__ long long s_min[8];
  const int q = wk.active_list[blockIdx.x];
  const QState& S = wk.qs[q];
  const int nh = S.nh, size = wk.split_size;
  const int t0 = size > 1 ? (int)((((int64_t)wk.split_rank - (int64_t)q * wk.TCAP) % size + size) % size) : 0;
  const float* cq = wk.cost32 + (int64_t)q * wk.HCAP;
  long long best = LLONG_MAX;
  for (int h = threadIdx.x; h < nh; h += blockDim.x) {
    if ((h / tile_h) % size != t0) continue;
    const long long key = ((long long)__float_as_uint(__ldcg(cq + h)) << 32) | (long long)h;
    best = min(best, key);
  }
  for (int o = 16; o > 0; o >>= 1) best = min(best, (long long)__shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long m = s_min[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = min(m, s_min[w]);
    keys[q] = m;
  }
}

// After the MIN all-reduce: the scan sees only the winning hypothesis (its
// cost; +inf for the rest of the batch), so the round runs at most one LO.
__global__ void __launch_bounds__(256) k_split_apply_argmin(Work wk, const long long* keys) {
  const int q = wk.active_list[blockIdx.x];
  const int nh = wk.qs[q].nh;
  const long long key = keys[q];
  const int hw = key == LLONG_MAX ? -1 : (int)(key & 0xffffffffLL);
  const float cw = __uint_as_float((unsigned)((unsigned long long)key >> 32));
  float* cq = wk.cost32 + (int64_t)q * wk.HCAP;
  for (int h = threadIdx.x; h < nh; h += blockDim.x) cq[h] = h == hw ? cw : CUDART_INF_F;
}

__global__ void k_fill_i64(long long* p, int n, long long v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

int launch_fill_i64(long long* p, int n, long long v, cudaStream_t st) {
  if (n <= 0) return 0;
  k_fill_i64<<<(n + 255) / 256, 256, 0, st>>>(p, n, v);
  return 1;
}

int launch_split_argmin(const Work& wk, int nactive, int num_sms, long long* keys, cudaStream_t st) {
  if (nactive <= 0) return 0;
  k_split_argmin<<<nactive, 256, 0, st>>>(wk, round_is_fine(wk, nactive, num_sms) ? kScoreTileHypsFine
                                                                                  : kScoreTileHyps, keys);
  return 1;
}

int launch_split_apply_argmin(const Work& wk, int nactive, const long long* keys, cudaStream_t st) {
  if (nactive <= 0) return 0;
  k_split_apply_argmin<<<nactive, 256, 0, st>>>(wk, keys);
  return 1;
}

// One round, kernel by kernel; `hook(stage, begin)` lets the caller bracket
// each launch with CUDA events (profiling) without touching the kernels.
// A/B knob VISLOC_CARVEOUT=1: every round kernel prefers the maximum shared
// memory carve-out, so consecutive (PDL-overlapped) kernels never need an
// L1 / shared-memory reconfiguration between them.
int carveout_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("VISLOC_CARVEOUT");
    mode = e ? atoi(e) : 0;
  }
  return mode;
}

static void set_round_carveouts() {
  static bool done[kMaxDevices] = {false};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (done[dev < kMaxDevices ? dev : 0]) return;
  done[dev < kMaxDevices ? dev : 0] = true;
  const int v = cudaSharedmemCarveoutMaxShared;
  cudaFuncSetAttribute(k_sample<256>, cudaFuncAttributePreferredSharedMemoryCarveout, v);
  cudaFuncSetAttribute(k_sample<1024>, cudaFuncAttributePreferredSharedMemoryCarveout, v);
  cudaFuncSetAttribute(k_p3p_roots, cudaFuncAttributePreferredSharedMemoryCarveout, v);
  cudaFuncSetAttribute(k_p3p_polish, cudaFuncAttributePreferredSharedMemoryCarveout, v);
  cudaFuncSetAttribute(k_compact<256>, cudaFuncAttributePreferredSharedMemoryCarveout, v);
  cudaFuncSetAttribute(k_compact<512>, cudaFuncAttributePreferredSharedMemoryCarveout, v);
  cudaFuncSetAttribute(k_compact<1024>, cudaFuncAttributePreferredSharedMemoryCarveout, v);
  cudaFuncSetAttribute(k_scan, cudaFuncAttributePreferredSharedMemoryCarveout, v);
}

int launch_round(const Work& wk, const Inputs& in, const RansacParams& p, int nactive, int num_sms,
                 cudaStream_t st, void (*hook)(void*, int, bool), void* hook_arg, int phase, int split) {
  if (carveout_mode()) set_round_carveouts();
  auto H = [&](int stage, bool begin) {
    if (hook) hook(hook_arg, stage, begin);
  };
  int n = 0;
  // scoring items: coarse (0), fine (1), or medium (2: 256-hypothesis tiles x
  // 4 splits, a single query's round — fewer, longer items; A/B VISLOC_MEDIUM=1: C4 6.55 vs 5.58 ms, off)
  static int medium = -1;
  if (medium < 0) {
    const char* e = getenv("VISLOC_MEDIUM");
    medium = e ? atoi(e) : 0;
  }
  const int fine = round_is_fine(wk, nactive, num_sms) ? (medium && nactive == 1 ? 2 : 1) : 0;
  const bool pdl = use_pdl(nactive) && !hook;  // (profiling brackets every launch with events)
  // split round (pruning on, coarse items, phase 0): head then rest (k_compact)
  const bool two = split && phase == 0 && wk.prune && !fine && kHeadHyps > 0;
  auto compact = [&](int mode) {
    H(kStageCompact, true);
    // threads per CTA (A/B knob VISLOC_COMPACT_NT: 256 / 512 / 1024); C3:
    // 256 -> 1.39 ms/step, 512 -> 1.63, 1024 -> 1.47 (spills at the 64-register
    // cap); a few queries (C4) take one 1024-thread pass: 2.3 vs 2.8 ms at 256
    static int cnt = -1;
    if (cnt < 0) {
      const char* e = getenv("VISLOC_COMPACT_NT");
      cnt = e ? atoi(e) : 256;
    }
    // up to 2 queries per SM (C5: 256, C4: 1): one 1024-thread pass per query
    // (C5 compact 0.096 -> 0.037 ms); big batches (C3: 1000) at 256 threads
    if (nactive <= 2 * num_sms) launch_k(k_compact<1024>, dim3(nactive), 1024, st, pdl, wk, fine, mode);
    else if (cnt == 256) launch_k(k_compact<256>, dim3(nactive), 256, st, pdl, wk, fine, mode);
    else if (cnt == 512) launch_k(k_compact<512>, dim3(nactive), 512, st, pdl, wk, fine, mode);
    else launch_k(k_compact<1024>, dim3(nactive), 1024, st, pdl, wk, fine, mode);
    H(kStageCompact, false);
    n += 1;
  };
  auto score = [&]() {
    H(kStageScore, true);
    n += launch_score(wk, (float)(p.tau * p.tau), num_sms, fine, nactive, st, pdl);  // (+ pruning tail)
    H(kStageScore, false);
  };
  auto scan = [&](int mode) {
    H(kStageScan, true);
    // function attributes are per device: set once for each device used
    // (host threads driving separate contexts may get here together)
    static int max_smem_dev[kMaxDevices] = {0};
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    int max_smem;
    {
      std::lock_guard<std::mutex> g(mu);
      int& ms = max_smem_dev[dev < kMaxDevices ? dev : 0];
      if (ms == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        v -= (int)(sizeof(LMShared<kScanThreads>) + 1024);  // static smem of the kernel
        cudaFuncSetAttribute(k_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
        ms = v;
      }
      max_smem = ms;
    }
    const size_t with_costs = kStageBytes + (size_t)wk.HCAP * sizeof(float);
    const int costs_smem = with_costs <= (size_t)max_smem ? 1 : 0;
    const size_t smem = costs_smem ? with_costs : kStageBytes;
    int cs = pick_cluster(nactive, VL_LO_MINB * num_sms);
    // a batch that fits the resident slots once but not twice (C5: 256 queries)
    // still gains from 2-CTA clusters: 1.97 -> 1.87 ms per C5 step (the
    // 1000-query C3 scan stays one CTA per query: clusters measured slower)
    if (cs == 1 && nactive <= VL_LO_MINB * num_sms) cs = 2;
    if (const char* e = getenv("VISLOC_SCAN_CS")) cs = atoi(e);  // tuning knob
    // (+ active-list compaction, except after a head phase)
    launch_clustered(k_scan, nactive, kScanThreads, smem, cs, st, pdl, wk, p, costs_smem, mode, fine);
    H(kStageScan, false);
    n += 1;
  };
  // phase 0: all; 1: up to the scores; 2: the scan; pipelined loop: 3: the
  // side chain (sampling + P3P), 4: the compaction, 5: scores + scan
  const bool side = phase == 0 || phase == 1 || phase == 3;
  const bool comp = phase == 0 || phase == 1 || phase == 4;
  const bool scr = phase == 0 || phase == 1 || phase == 5;
  const bool scn = phase == 0 || phase == 2 || phase == 5;
  if (side) {
    H(kStageSample, true);
    if (nactive * 4 <= num_sms) launch_k(k_sample<1024>, dim3(nactive), 1024, st, pdl, wk, p);
    else launch_k(k_sample<256>, dim3(nactive), 256, st, pdl, wk, p);
    H(kStageSample, false);
    H(kStageP3P, true);
    dim3 gr(nactive, (wk.B + kP3PRootThreads - 1) / kP3PRootThreads);
    launch_k(k_p3p_roots, gr, kP3PRootThreads, st, pdl, wk, in);
    dim3 gp(nactive, (wk.B + kP3PThreads - 1) / kP3PThreads);
    launch_k(k_p3p_polish, gp, kP3PThreads, st, pdl, wk);
    H(kStageP3P, false);
    n += 3;
  }
  if (two) {
    compact(1);
    score();
    scan(1);
    compact(2);
  } else if (comp) {
    compact(0);
  }
  if (scr) score();
  if (scn) scan(two ? 2 : 0);
  return n;
}

// ------------------------------------------------------------------ final stage
constexpr int kFinalThreads = VL_LO_NT;

// Full-set MSAC pass (posest.py:160-175 / 284-299) of a one-CTA query with
// the caller's px / X / w arrays streamed through the TMA ring: chunk c is
// the 512 points [a0 + 512 c, ...) of the global arrays, a0 = S.off rounded
// down to even so every bulk copy (px 16 B, X 24 B, w 8 B per point) starts
// and ends on a 16-B boundary; a trailing odd point is read directly.  The
// plain-load pass was latency bound (ncu, C5: long_scoreboard 42 % of the
// k_final stalls at 13 warps/SM).  With COMPACT the ordered inlier
// compaction X[flags_full] (posest.py:291-294) is done in the same pass from
// the staged records: one block scan of (first-half, second-half) flag
// counts packed into an int per chunk, so the inliers are not re-read.
// Returns cost / count in sm.red[0..1] like msac_pass.
constexpr int kAosSlotPx = 0, kAosSlotX = kStageCh * 16, kAosSlotW = kStageCh * 40;  // byte offsets in a slot

__device__ __forceinline__ void aos_issue(const double* px, const double* X, const double* w, int64_t a0, int64_t e,
                                          unsigned char* ring, uint64_t* bars, int c) {
  const int slot = c % kStageN;
  const int64_t s = a0 + (int64_t)c * kStageCh;
  const unsigned m = (unsigned)(e - s < kStageCh ? e - s : kStageCh);
  unsigned char* dst = ring + (size_t)slot * kStageCh * 48;
  const unsigned bar = smem_u32(bars + slot);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(m * 48u) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst + kAosSlotPx)), "l"(px + 2 * s), "r"(m * 16u), "r"(bar) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst + kAosSlotX)), "l"(X + 3 * s), "r"(m * 24u), "r"(bar) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst + kAosSlotW)), "l"(w + s), "r"(m * 8u), "r"(bar) : "memory");
}

template <int NT, bool COMPACT>
__device__ void msac_full_staged(LMShared<NT>& sm, const Inputs& in, int64_t g0, int n, const Intr& cin, double tau,
                                 uint8_t* flags, double2* cpk, unsigned char* ring, uint64_t* bars, int* warp_tot,
                                 int direct) {
  static_assert(kStageCh == 2 * NT, "two points per thread per chunk");
  const double t2 = dmul(tau, tau);
  double R[9], t[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = sm.R[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = sm.t[k];
  const int64_t g1 = g0 + n, a0 = g0 & ~(int64_t)1, e = g1 & ~(int64_t)1;
  const int nch = (int)((e - a0 + kStageCh - 1) / kStageCh);
  if (threadIdx.x == 0) {
    for (int b = 0; b < kStageN; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + b)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int c = 0; c < min(kStageN, nch); ++c) aos_issue(in.px, in.X, in.w, a0, e, ring, bars, c);
  double acc[2] = {0.0, 0.0};
  int running = 0;
  auto point = [&](int64_t gi, const double* P, double u, double v, double w, int& f) {
    const double e2 = msac_e2(R, t, cin, P, u, v);
    acc[0] = acc[0] + dmul(w, fmin(e2, t2));
    f = e2 < t2 ? 1 : 0;
    acc[1] += (double)f;
    flags[gi - g0] = (uint8_t)f;
  };
  for (int c = 0; c < nch; ++c) {
    const unsigned bar = smem_u32(bars + c % kStageN);
    const unsigned parity = (unsigned)(c / kStageN) & 1u;
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITA_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITA_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
    const unsigned char* buf = ring + (size_t)(c % kStageN) * kStageCh * 48;
    const double2* spx = reinterpret_cast<const double2*>(buf + kAosSlotPx);
    const double* sX = reinterpret_cast<const double*>(buf + kAosSlotX);
    const double* sw = reinterpret_cast<const double*>(buf + kAosSlotW);
    const int64_t s = a0 + (int64_t)c * kStageCh;
    const int m = (int)(e - s < kStageCh ? e - s : kStageCh);
    double P[2][3], u[2], v[2], w[2];
    int f[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = threadIdx.x + h * NT;
      if (j < m && s + j >= g0) {
        if (direct) {
          const int64_t gi = s + j;
          P[h][0] = in.X[3 * gi];
          P[h][1] = in.X[3 * gi + 1];
          P[h][2] = in.X[3 * gi + 2];
          u[h] = in.px[2 * gi];
          v[h] = in.px[2 * gi + 1];
          w[h] = in.w[gi];
        } else {
        const double2 q = spx[j];
        P[h][0] = sX[3 * j];
        P[h][1] = sX[3 * j + 1];
        P[h][2] = sX[3 * j + 2];
        u[h] = q.x;
        v[h] = q.y;
        w[h] = sw[j];
        }
        point(s + j, P[h], u[h], v[h], w[h], f[h]);
      }
    }
    if constexpr (COMPACT) {
      int total;
      const int ex = block_excl_scan<NT>(f[0] | (f[1] << 16), warp_tot, total);
      const int t0 = total & 0xffff;
      if (f[0]) pack_point(cpk, running + (ex & 0xffff), P[0], u[0], v[0], w[0]);
      if (f[1]) pack_point(cpk, running + t0 + (ex >> 16), P[1], u[1], v[1], w[1]);
      running += t0 + (total >> 16);
    } else {
      __syncthreads();  // every thread is done with the slot before it is refilled
    }
    if (threadIdx.x == 0 && c + kStageN < nch) aos_issue(in.px, in.X, in.w, a0, e, ring, bars, c + kStageN);
  }
  stage_inval(bars);
  if (g1 != e && threadIdx.x == 0) {  // odd end: the last point, after every staged one
    const int64_t gi = g1 - 1;
    double P[3] = {in.X[3 * gi], in.X[3 * gi + 1], in.X[3 * gi + 2]};
    int f = 0;
    point(gi, P, in.px[2 * gi], in.px[2 * gi + 1], in.w[gi], f);
    if (COMPACT && f) pack_point(cpk, running, P, in.px[2 * gi], in.px[2 * gi + 1], in.w[gi]);
  }
  block_sum<NT, 2>(acc, sm.scratch, sm.red);
}

__global__ void __launch_bounds__(kFinalThreads, VL_LO_MINB) k_final(Work wk, Inputs in, Outputs out, RansacParams p,
                                                         int q_base, int staged) {
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ uint64_t stage_bar[kStageN];
  __shared__ LMShared<kFinalThreads> sm;
  __shared__ int warp_tot[32];
  const unsigned cr = cl_rank(), cs = cl_size();
  const int q = blockIdx.x / cs;
  const QState& S = wk.qs[q];
  const int64_t gq = q_base + q;
  const int n = S.n;
  uint8_t* flags = out.flags + S.off;
  const AosPts full{in.px + 2 * S.off, in.X + 3 * S.off, in.w + S.off, n};
  const Intr cin = S.in;
  auto write_small = [&](const Pose& ps, int64_t cnt, double score, int conv) {
    if (threadIdx.x == 0 && cr == 0) {
      for (int i = 0; i < 4; ++i) out.q[4 * gq + i] = ps.q[i];
      for (int i = 0; i < 3; ++i) out.t[3 * gq + i] = ps.t[i];
      out.inlier_count[gq] = cnt;
      out.score[gq] = score;
      out.iterations[gq] = S.iters;
      out.converged[gq] = conv;
      if (out.stats) {
        out.stats[4 * gq + 0] = S.lo_calls;
        out.stats[4 * gq + 1] = S.hyps;
        out.stats[4 * gq + 2] = S.evals;
        out.stats[4 * gq + 3] = S.rounds;
      }
    }
  };
  if (!S.has_best) {
    for (int i = threadIdx.x + kFinalThreads * cr; i < n; i += kFinalThreads * cs) flags[i] = 0;
    Pose id;
    id.q[0] = 1;
    id.q[1] = id.q[2] = id.q[3] = 0;
    id.t[0] = id.t[1] = id.t[2] = 0;
    write_small(id, 0, CUDART_INF, 0);
    return;
  }
  const Pose best = S.best;
  set_eval_pose(sm, best);
  double2* cpk = wk.comp_pk + 3 * S.coff;
  if (staged & 1)  // one CTA per query: TMA-streamed pass with the inlier compaction fused
    msac_full_staged<kFinalThreads, true>(sm, in, S.off, n, cin, p.tau, flags, cpk, dyn_smem, stage_bar, warp_tot,
                                          staged & 4);
  else
    msac_pass<kFinalThreads>(sm, full, cin, p.tau, flags);  // cluster-wide; flags visible after its cluster barrier
  const double cost_full = sm.red[0];
  const int64_t cnt_full = (int64_t)sm.red[1];
  if (cnt_full < 3) {
    write_small(best, cnt_full, cost_full, 0);
    return;
  }
  if (!(staged & 1)) {
  // ordered compaction of the full-set inliers (X[flags_full], posest.py:291-294):
  // CTA r of the cluster owns the contiguous range [lo, hi) of the point list
  __syncthreads();
  const int lo = (int)((int64_t)n * cr / cs), hi = (int)((int64_t)n * (cr + 1) / cs);
  int mine = 0;
  for (int i = lo + threadIdx.x; i < hi; i += kFinalThreads) mine += flags[i] ? 1 : 0;
  {
    double c[1] = {(double)mine};
    block_sum<kFinalThreads, 1>(c, sm.scratch, sm.red2);
  }
  if (threadIdx.x == 0) sm.cnt[0] = (long long)sm.red2[0];
  int start = 0;
  if (cs > 1) {
    cl_sync();
    for (unsigned r = 0; r < cr; ++r) start += (int)cl_load_ll(&sm.cnt[0], r);
  }
  int running = start;
  for (int base = lo; base < hi; base += kFinalThreads) {
    const int i = base + threadIdx.x;
    const int f = (i < hi && flags[i]) ? 1 : 0;
    int total;
    const int ex = block_excl_scan<kFinalThreads>(f, warp_tot, total);
    if (f) {
      double P[3], u, v, w;
      full.load(i, P, u, v, w);
      pack_point(cpk, running + ex, P, u, v, w);
    }
    running += total;
  }
  }
  __threadfence();
  asm volatile("fence.proxy.async.global;" ::: "memory");  // compacted records are read back by TMA
  __syncthreads();
  if (cs > 1) cl_sync();  // compacted points of every CTA visible cluster-wide
  const StagedPts inl{cpk, (int)cnt_full, reinterpret_cast<double2*>(dyn_smem), stage_bar};
  lm_refine<kFinalThreads>(sm, inl, cin, best, kCauchy, p.cauchy, p.lm_max_iters, 1e-10, 1e-12, nullptr,
                           nullptr);
  const Pose fin = sm.cur;
  set_eval_pose(sm, fin);
  if (staged & 2)
    msac_full_staged<kFinalThreads, false>(sm, in, S.off, n, cin, p.tau, flags, nullptr, dyn_smem, stage_bar, warp_tot,
                                           staged & 4);
  else
    msac_pass<kFinalThreads>(sm, full, cin, p.tau, flags);
  write_small(fin, (int64_t)sm.red[1], sm.red[0], 1);
}

int launch_final(const Work& wk, const Inputs& in, const Outputs& out, const RansacParams& p, int Q,
                 int q_base, cudaStream_t st) {
  static bool attr_dev[kMaxDevices] = {false};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(mu);
    bool& attr = attr_dev[dev < kMaxDevices ? dev : 0];
    if (!attr) {  // the staging ring needs more than the 48 KB default dynamic smem (per device)
      cudaFuncSetAttribute(k_final, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStageBytes);
      attr = true;
    }
  }
  int cs = pick_cluster(Q, VL_LO_MINB * 148);
  if (const char* e = getenv("VISLOC_FINAL_CS")) cs = atoi(e);  // tuning knob
  // TMA-streamed full-set passes need one CTA per query and 16-B aligned arrays
  int staged = cs == 1 && ((reinterpret_cast<uintptr_t>(in.px) | reinterpret_cast<uintptr_t>(in.X) |
                            reinterpret_cast<uintptr_t>(in.w)) & 15) == 0;
  if (staged) staged = 3;  // bit 0: first pass + fused compaction, bit 1: final pass, bit 2: debug (global reads)
  if (const char* e = getenv("VISLOC_FINAL_STAGED")) staged = staged ? atoi(e) : 0;  // A/B knob
  launch_clustered(k_final, Q, kFinalThreads, kStageBytes, cs, st, false, wk, in, out, p, q_base, staged);
  return 1;
}

// ------------------------------------------------------------------ standalone msac / refine
__global__ void __launch_bounds__(512) k_msac(Pose pose, AosPts ps, Intr in, double tau, double* red_out,
                                              uint8_t* flags) {
  __shared__ LMShared<512> sm;
  set_eval_pose(sm, pose);
  msac_pass<512>(sm, ps, in, tau, flags);
  if (threadIdx.x == 0) {
    red_out[0] = sm.red[0];
    red_out[1] = sm.red[1];
  }
}

int launch_msac(const Pose& pose, const double* px, const double* X, const double* w, int n, Intr in,
                double tau, double* red_out, uint8_t* flags, cudaStream_t st) {
  k_msac<<<1, 512, 0, st>>>(pose, AosPts{px, X, w, n}, in, tau, red_out, flags);
  return 1;
}

__global__ void __launch_bounds__(512) k_refine(Pose start, AosPts ps, Intr in, int kind, double scale,
                                                int max_iters, double gtol, double ctol, Pose* pose_out,
                                                int* info_out, double* trace) {
  __shared__ LMShared<512> sm;
  int tl = 0;
  LMResult r = lm_refine<512>(sm, ps, in, start, kind, scale, max_iters, gtol, ctol, trace, &tl);
  if (threadIdx.x == 0) {
    *pose_out = sm.cur;
    info_out[0] = r.converged;
    info_out[1] = r.iterations;
    info_out[2] = tl;
  }
}

int launch_refine(const Pose& start, const double* px, const double* X, const double* w, int n, Intr in,
                  int kind, double scale, int max_iters, double gtol, double ctol, Pose* pose_out,
                  int* info_out, double* trace, cudaStream_t st) {
  k_refine<<<1, 512, 0, st>>>(start, AosPts{px, X, w, n}, in, kind, scale, max_iters, gtol, ctol,
                              pose_out, info_out, trace);
  return 1;
}

// robust_cost (refine.py:135-149): one fused cost pass.
__global__ void __launch_bounds__(512) k_robust_cost(Pose pose, AosPts ps, Intr in, int kind, double scale,
                                                     double* out) {
  __shared__ LMShared<512> sm;
  set_eval_pose(sm, pose);
  lm_pass<512, false>(sm, ps, in, kind, scale);
  if (threadIdx.x == 0) out[0] = sm.red[0];
}

int launch_robust_cost(const Pose& pose, const double* px, const double* X, const double* w, int n, Intr in,
                       int kind, double scale, double* out, cudaStream_t st) {
  k_robust_cost<<<1, 512, 0, st>>>(pose, AosPts{px, X, w, n}, in, kind, scale, out);
  return 1;
}

// pose_residuals + pose_jacobian (refine.py:90-132): per-point residual,
// camera z and the analytic 2x6 Jacobian (rows zeroed at/behind the camera).
__global__ void k_residuals(Pose pose, const double* px, const double* X, int n, Intr in, double* res,
                            double* z_out, double* J) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double R[9];
  q2R(pose.q, R);
  const double P[3] = {X[3 * i], X[3 * i + 1], X[3 * i + 2]};
  double x, y, z;
  cam_point(R, pose.t, P, x, y, z);
  const double u = dadd(__ddiv_rn(dmul(in.fx, x), z), in.cx);
  const double v = dadd(__ddiv_rn(dmul(in.fy, y), z), in.cy);
  if (res) {
    res[2 * i] = dsub(u, px[2 * i]);
    res[2 * i + 1] = dsub(v, px[2 * i + 1]);
  }
  if (z_out) z_out[i] = z;
  if (J) {
    double* Ji = J + 12 * (int64_t)i;
    if (!(z > 0)) {
      for (int k = 0; k < 12; ++k) Ji[k] = 0.0;
      return;
    }
    const double p00 = in.fx / z, p02 = -in.fx * x / (z * z);
    const double p11 = in.fy / z, p12 = -in.fy * y / (z * z);
    Ji[0] = p02 * y;
    Ji[1] = p00 * z + p02 * (-x);
    Ji[2] = p00 * (-y);
    Ji[3] = p00;
    Ji[4] = 0.0;
    Ji[5] = p02;
    Ji[6] = p11 * (-z) + p12 * y;
    Ji[7] = p12 * (-x);
    Ji[8] = p11 * x;
    Ji[9] = 0.0;
    Ji[10] = p11;
    Ji[11] = p12;
  }
}

int launch_residuals(const Pose& pose, const double* px, const double* X, int n, Intr in, double* res, double* z,
                     double* J, cudaStream_t st) {
  if (n <= 0) return 0;
  k_residuals<<<(n + 255) / 256, 256, 0, st>>>(pose, px, X, n, in, res, z, J);
  return 1;
}

}  // namespace vl
