// fp32 MSAC hypothesis scoring — kernel template (see vl_score.cu).
#pragma once
#include "vl_internal.h"

namespace vl {

// resident CTAs per SM of the coarse scorer (vl_score.cu)
#ifndef VL_SCORE_MINB
#define VL_SCORE_MINB 3
#endif

// ---------------------------------------------------------------- f32x2 path
// Blackwell packed FP32 (FFMA2 / FMUL2): one instruction evaluates the same
// step for TWO CORRESPONDENCES of one hypothesis.  Records are stored in
// pairs (SoA float2: X, Y, Z, cx-u, cy-v, w of points 2k and 2k+1), the
// hypothesis' fx/fy-folded [R|t] entries are scalars broadcast to both halves
// (SASS `Rn.F32`).  Consecutive FFMA2 of the HT hypotheses of a thread then
// share the record operand (register reuse cache), which halves the
// register-file reads per instruction against the earlier packing (two
// hypotheses x one broadcast coordinate): tools/score_mix_bench.cu measured
// 2.255e12 vs 1.982e12 evaluations/s for the same 14 FFMA2/FMUL2 + 2 MUFU +
// 4 FMNMX per pair of evaluations.
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __ffma2_rn(a, b, make_float2(-0.f, -0.f)); }

__device__ __forceinline__ float rcp_approx_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// r = 1 / max(z, 0): +inf for z <= 0 (behind camera / on the camera plane),
// so e2 becomes inf or NaN and fminf (IEEE minNum) maps it to tau^2.  The
// clamp runs on the ALU pipe, the reciprocal on the MUFU pipe: the FMA pipe
// only sees the 14 FFMA2/FMUL2 of the evaluation pair.  A padding record
// (odd subset size) has w = 0 and adds +0.
#ifdef VL_SCORE_DIV_RN
// A/B variant (not the product): IEEE-rounded quotients x / z, y / z as the
// reference computes them (posest.py:209-211), for the cost / speed comparison
// quoted in DESIGN.md
#define VL_SCORE_DU_DV(x_, y_, z_)                                                                \
  const float2 zc_ = make_float2(fmaxf(z_.x, 0.f), fmaxf(z_.y, 0.f));                             \
  const float2 du_ = make_float2(__fadd_rn(__fdiv_rn(x_.x, zc_.x), A2.x), __fadd_rn(__fdiv_rn(x_.y, zc_.y), A2.y)); \
  const float2 dv_ = make_float2(__fadd_rn(__fdiv_rn(y_.x, zc_.x), B2.x), __fadd_rn(__fdiv_rn(y_.y, zc_.y), B2.y));
#else
#define VL_SCORE_DU_DV(x_, y_, z_)                                                                \
  const float2 r_ = make_float2(rcp_approx_ftz(fmaxf(z_.x, 0.f)), rcp_approx_ftz(fmaxf(z_.y, 0.f))); \
  const float2 du_ = fma2(x_, r_, A2);                                                            \
  const float2 dv_ = fma2(y_, r_, B2);
#endif
#define VL_SCORE_EVAL2(Ph, acch)                                                                  \
  {                                                                                               \
    const float2 x_ = fma2(X2, f2(Ph[0]), fma2(Y2, f2(Ph[1]), fma2(Z2, f2(Ph[2]), f2(Ph[3]))));   \
    const float2 y_ = fma2(X2, f2(Ph[4]), fma2(Y2, f2(Ph[5]), fma2(Z2, f2(Ph[6]), f2(Ph[7]))));   \
    const float2 z_ = fma2(X2, f2(Ph[8]), fma2(Y2, f2(Ph[9]), fma2(Z2, f2(Ph[10]), f2(Ph[11])))); \
    VL_SCORE_DU_DV(x_, y_, z_)                                                                    \
    float2 e2_ = fma2(du_, du_, mul2(dv_, dv_));                                                  \
    e2_.x = fminf(e2_.x, tau2);                                                                   \
    e2_.y = fminf(e2_.y, tau2);                                                                   \
    acch = fma2(W2, e2_, acch);                                                                   \
  }

// Work item = (query, tile of NT*HT hypotheses, ns <= SPI consecutive
// correspondence splits of SCH records).  The canonical fp32 cost of a
// hypothesis is  sum over split groups (in order) of the group sum
// ((p0 + p1) + p2) + p3  of its splits' record sums, a split's sum being
// (even records, in order) + (odd records, in order) — every
// split is accumulated by exactly one thread in record order, so neither the
// tile shape (HT), the splits per item (SPI) nor the grid changes a single
// bit.  The last item to finish a (query, tile) — atomic ticket per tile —
// reduces the tile's partial slots in that order and writes the final costs.
template <int NT, int HT, int SPI, int SCH>
constexpr size_t score_smem_bytes() {
  return sizeof(float4) * (3 * SPI * SCH / 2) + sizeof(float) * SPI * (SPI > 1 ? NT * HT : 1);
}

// The closing item of a (query, tile): canonical sums of the tile's
// hypotheses from the partial slots (and, in pruned rounds, the survivor list
// for k_score_tail).  PRUNE = false is the kernel instance of runs without
// pruning, so the pruning code's registers stay out of it (-2 % scoring time,
// 161 vs 168 registers); the pruning instance calls it out of line (-1 %).
#ifndef VL_CLOSE_FINE_G
#define VL_CLOSE_FINE_G 8  // fine closer: split groups loaded per batch (A/B, C4 ms: 4 8.79, 8 8.72, 20 9.17)
#endif
template <int NT, int HT, int SPI, int SCH, bool PRUNE>
__device__ __forceinline__ void score_close_tile(const Work& wk, const ScoreItem& item, const float* outq, int tile0,
                                               float* red_area, int* sh) {
  const QState& S = wk.qs[item.q];
  const int nh = S.h_hi, nsub = S.nsub;
  const int NS = S.nsplit;
  const int NG = (NS + kGroupSplits - 1) / kGroupSplits;
  __threadfence();
  const int h1 = min(nh, tile0 + NT * HT);
  float* costq = wk.cost32 + (int64_t)item.q * wk.HCAP;
  // pruned round: the tile holds the group sums of splits [0, sA) (the last
  // group possibly partial: the left fold of its first sA mod 4 splits);
  // their running sum is a lower bound of the final fp32 cost (every later
  // term and split sum is >= 0, fp32 addition is monotone and the group sum
  // is a left fold).  A hypothesis whose bound is >= the best cost can never
  // be accepted by the ordered scan (`cost < best`, posest.py:258), so the
  // bound stands as its cost; the others are listed for k_score_tail
  const int gend = SPI == 1 ? NG : (S.sA + kGroupSplits - 1) / kGroupSplits;
  const bool pruning = PRUNE && SPI > 1 && S.sA < NS;
  const double best = S.best_cost;
  // a tile's surviving hypotheses (pruned rounds), in the split-sum area
  // (coarse items: SPI * NT * HT floats >= NT * HT), free once the ticket is taken
  int* s_surv = reinterpret_cast<int*>(red_area);
  if (pruning) {
    if (threadIdx.x == 0) sh[0] = 0;
    __syncthreads();
  }
  for (int h = tile0 + threadIdx.x; h < h1; h += NT) {
    // the partials of 4 groups (fine: 16 splits) / 8 groups (coarse) are
    // loaded before they are added, in the canonical order, so the
    // closing item waits for a few L2 round trips instead of one per group
    float c = 0.f;
    if (SPI == 1) {
      for (int g0 = 0; g0 < NG; g0 += VL_CLOSE_FINE_G) {
        float v[VL_CLOSE_FINE_G][kGroupSplits];
#pragma unroll
        for (int gg = 0; gg < VL_CLOSE_FINE_G; ++gg)
#pragma unroll
          for (int k = 0; k < kGroupSplits; ++k) {
            const int sp = (g0 + gg) * kGroupSplits + k;
            v[gg][k] = sp < NS ? __ldcg(outq + (int64_t)sp * wk.HCAP + h) : 0.f;
          }
#pragma unroll
        for (int gg = 0; gg < VL_CLOSE_FINE_G; ++gg) {
          const int g = g0 + gg;
          if (g < NG) {
            float gs = v[gg][0];
#pragma unroll
            for (int k = 1; k < kGroupSplits; ++k)
              if (g * kGroupSplits + k < NS) gs += v[gg][k];
            c += gs;
          }
        }
      }
    } else {
      for (int g0 = 0; g0 < gend; g0 += 8) {
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = g0 + k < gend ? __ldcg(outq + (int64_t)(g0 + k) * wk.HCAP + h) : 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (g0 + k < gend) c += v[k];
      }
    }
    costq[h] = c;
    if (pruning && !((double)c >= best)) s_surv[atomicAdd(&sh[0], 1)] = h;
  }
  if (pruning) {
    // append the tile's survivors to the query's list; the query's last
    // tile to close turns the list into tail tasks of up to 32 hypotheses
    QState* Sq = wk.qs + item.q;
    __syncthreads();
    const int ns_ = sh[0];
    if (threadIdx.x == 0) sh[1] = ns_ ? atomicAdd(&Sq->nsurv, ns_) : 0;
    __syncthreads();
    int* sv = wk.surv + (int64_t)item.q * wk.HCAP;
    for (int i = threadIdx.x; i < ns_; i += NT) sv[sh[1] + i] = s_surv[i];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long rest = (long long)nsub - min((long long)nsub, (long long)S.sA * SCH);
      atomicAdd(wk.prune_ctr, (unsigned long long)((h1 - tile0 - ns_) * rest));
      atomicAdd(wk.prune_ctr + 1, (unsigned long long)(ns_ * rest));
      const int ntile = (nh - S.h_lo + NT * HT - 1) / (NT * HT);
      if (atomicAdd(&Sq->tiles_closed, 1) == ntile - 1) {
        __threadfence();
        const int nq = atomicAdd(&Sq->nsurv, 0), ntask = (nq + 31) / 32;
        const int base = ntask ? atomicAdd(wk.item_count + 3, ntask) : 0;
        for (int k = 0; k < ntask; ++k)
          if (base + k < wk.tail_cap) wk.tail[base + k] = TailTask{item.q, 32 * k, min(32, nq - 32 * k), 0};
      }
    }
  }
}

template <int NT, int HT, int SPI, int SCH>
__device__ __noinline__ void score_close_tile_pruning(const Work& wk, const ScoreItem& item, const float* outq,
                                                      int tile0, float* red_area, int* sh) {
  score_close_tile<NT, HT, SPI, SCH, true>(wk, item, outq, tile0, red_area, sh);
}

// Register cap of the scorer via __maxnreg__ (A/B knob; 0 =
// __launch_bounds__(NT, MINB) alone, 159 registers with the hsrc row reads):
// C3 / C3 pruned ms per step 93.3 / 48.5 uncapped, 93.5 / 48.7 at 160 (154
// registers), 94.0 at 152.
#ifndef VL_SCORE_MAXNREG
#define VL_SCORE_MAXNREG 0
#endif
#if VL_SCORE_MAXNREG > 0
// (the fine instance keeps its occupancy bound: 65536 / (NT x MINB) rounded down to 8)
#define VL_SCORE_BOUNDS(NT, MINB) __maxnreg__((MINB) == VL_SCORE_MINB ? VL_SCORE_MAXNREG : 65536 / ((NT) * (MINB)) / 8 * 8)
#else
#define VL_SCORE_BOUNDS(NT, MINB) __launch_bounds__(NT, MINB)
#endif
template <int NT, int HT, int SPI, int SCH, int MINB, int UNR, bool PRUNE>
__global__ void VL_SCORE_BOUNDS(NT, MINB) k_score2_t(Work wk, float tau2) {
  pdl_enter();
  static_assert(SCH % 2 == 0, "splits hold whole record pairs");
  constexpr int NW = NT / 32;
  constexpr int WHYP = 32 * HT;  // hypotheses per warp slice
  static_assert(SPI == 1 || SPI == kGroupSplits, "coarse items are exactly one split group");
  // record pairs (X2, Y2), (Z2, A2), (B2, W2) in dynamic smem (can exceed the
  // 48 KB static limit for 8-split items), split sums of coarse items after them
  extern __shared__ __align__(16) unsigned char score_dyn[];
  float4* rec = reinterpret_cast<float4*>(score_dyn);                                   // [3 * SPI * SCH / 2]
  float (*red)[SPI > 1 ? NT * HT : 1] = reinterpret_cast<float (*)[SPI > 1 ? NT * HT : 1]>(
      score_dyn + sizeof(float4) * (3 * SPI * SCH / 2));                                // [SPI][NT * HT]
  __shared__ int s_it, s_last, s_sh[2];
  const int nitems = wk.item_count[0];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // dynamic work cursor: items differ in cost (partial tiles), and a static
  // grid stride can alias with the per-query item period
  while (true) {
    if (threadIdx.x == 0) s_it = atomicAdd(&wk.item_count[1], 1);
    __syncthreads();
    const int it = s_it;
    if (it >= nitems) break;
    const ScoreItem item = wk.items[it];
    const QState& S = wk.qs[item.q];
    const int nh = S.h_hi, nsub = S.nsub;  // this phase's hypotheses end at h_hi; tiles count from h_lo
    const int tile0 = S.h_lo + item.tile * (NT * HT);
    const int ns = item.nsplit;
    float* outq = wk.partial + (int64_t)item.q * wk.NSPLIT * wk.HCAP;
    // partial slot layout: fine items (SPI == 1) write one slot per split;
    // coarse items write one slot per group of kGroupSplits splits, holding
    // the group sum ((p0 + p1) + p2) + p3 that k_scan forms itself in fine mode
    const int c0 = item.split * SCH;
    const int cn = min(ns * SCH, nsub - c0);
    const int pn = (cn + 1) >> 1;  // record pairs (the last one padded when nsub is odd)
    const float4* src = wk.sub32 + 3 * ((S.sub_off + c0) >> 1);
    // A partially filled (last) tile of r hypotheses needs WH = ceil(r / WHYP)
    // warp slices; the other warps take other splits of the item (G groups),
    // so a short tile does not leave warps idle.
    const int r = min(NT * HT, nh - tile0);
    const int WH = (r + WHYP - 1) / WHYP;
    const int G = NW / WH;
    const int hs = w % WH, grp = w / WH;
    __syncthreads();
    for (int k = threadIdx.x; k < 3 * pn; k += NT) rec[k] = src[k];
    float P[HT][12];
    // hypotheses hid0 .. hid0 + HT - 1 of this thread (thread-contiguous)
    const int hid0 = tile0 + hs * WHYP + lane * HT;
#if VL_P32_COPY
    const float* Pq = wk.P32 + (int64_t)item.q * 12 * wk.HCAP;
#pragma unroll
    for (int j = 0; j < HT; ++j) {
      const int h = hid0 + j < nh ? hid0 + j : 0;
#pragma unroll
      for (int c = 0; c < 12; ++c) P[j][c] = Pq[(int64_t)c * wk.HCAP + h];
    }
#else
    // hypothesis h's row at its solution slot column hsrc[h] (k_p3p_polish)
    const float* Pq = (wk.P32s ? wk.P32s : wk.P32) + (int64_t)item.q * 12 * wk.HCAP;
    const int* hq = wk.hsrc + (int64_t)item.q * wk.HCAP;
#pragma unroll
    for (int j = 0; j < HT; ++j) {
      const int col = wk.P32s ? __ldg(hq + (hid0 + j < nh ? hid0 + j : 0)) : (hid0 + j < nh ? hid0 + j : 0);
#pragma unroll
      for (int c = 0; c < 12; ++c) P[j][c] = Pq[(int64_t)c * wk.HCAP + col];
    }
#endif
    __syncthreads();
    for (int s = grp; s < ns && grp < G; s += G) {
      float2 acc[HT];
#pragma unroll
      for (int j = 0; j < HT; ++j) acc[j] = make_float2(0.f, 0.f);
      const int pb = s * (SCH / 2), pe = min(pb + SCH / 2, pn);
#pragma unroll UNR
      for (int c = pb; c < pe; ++c) {
        const float4 r0 = rec[3 * c], r1 = rec[3 * c + 1], r2 = rec[3 * c + 2];
        const float2 X2 = make_float2(r0.x, r0.y), Y2 = make_float2(r0.z, r0.w);
        const float2 Z2 = make_float2(r1.x, r1.y), A2 = make_float2(r1.z, r1.w);
        const float2 B2 = make_float2(r2.x, r2.y), W2 = make_float2(r2.z, r2.w);
#pragma unroll
        for (int j = 0; j < HT; ++j) VL_SCORE_EVAL2(P[j], acc[j]);
      }
      // the split's sum: even records + odd records
      if (SPI == 1) {
        float* out = outq + (int64_t)(item.split + s) * wk.HCAP;
#pragma unroll
        for (int j = 0; j < HT; ++j)
          if (hid0 + j < nh) out[hid0 + j] = acc[j].x + acc[j].y;
      } else {
        // park the split sum in smem (no per-thread group accumulator stays
        // live across the record loop); the group sum is formed below
#pragma unroll
        for (int j = 0; j < HT; ++j) red[s][hs * WHYP + lane * HT + j] = acc[j].x + acc[j].y;
      }
    }
    if (SPI > 1) {
      float* out = outq + (int64_t)(item.split / kGroupSplits) * wk.HCAP;
      if (G > 1) __syncthreads();  // splits of a partial tile came from other warp groups
      if (grp == 0) {
#pragma unroll
        for (int j = 0; j < HT; ++j) {
          float sx = red[0][hs * WHYP + lane * HT + j];  // ((p0 + p1) + p2) + p3, in split order
          for (int s = 1; s < ns; ++s) sx += red[s][hs * WHYP + lane * HT + j];
          if (hid0 + j < nh) out[hid0 + j] = sx;
        }
      }
    }
    // ---- tile completion ticket (threadfence reduction pattern)
    __threadfence();
    __syncthreads();
    const int NS = S.nsplit;
    if (threadIdx.x == 0) {
      // coarse: the groups of splits [0, sA) (sA < NS in pruned rounds)
      const int tile_items = SPI == 1 ? NS : (S.sA + kGroupSplits - 1) / kGroupSplits;
      s_last = atomicAdd(wk.tile_cnt + (int64_t)item.q * wk.TCAP + item.tile, 1) == tile_items - 1;
    }
    __syncthreads();
    if (s_last) {
      if constexpr (PRUNE) score_close_tile_pruning<NT, HT, SPI, SCH>(wk, item, outq, tile0, &red[0][0], s_sh);
      else score_close_tile<NT, HT, SPI, SCH, false>(wk, item, outq, tile0, &red[0][0], s_sh);
    }
  }
}

// Scoring tail of a pruned round: one CTA per task (up to 32 surviving
// hypotheses of one query), lane = hypothesis, warp w = split w of the
// current split group.  Each survivor's canonical sum is rebuilt from the
// tile's group slots in the canonical order (full groups of [0, sA), then
// the left fold of the partial group, continued), and completed over the
// remaining splits: a group's 512 records are staged in shared memory (one
// cooperative load, broadcast reads), every warp forms its split sum with the
// same EVAL2 sequence as k_score2_t, and warp 0 folds the group sums
// ((p0 + p1) + p2) + p3 into the running sum — so the cost bits equal a full
// scoring.
template <int NT>
__global__ void __launch_bounds__(NT) k_score_tail(Work wk, float tau2) {
  pdl_enter();
  static_assert(NT / 32 == kGroupSplits, "one warp per split of a group");
  constexpr int GP = kGroupSplits * kScoreChunk / 2;  // record pairs per group
  __shared__ __align__(16) float4 rec[3 * GP];
  __shared__ float red[kGroupSplits][32];
  const int ntask = min((int64_t)wk.item_count[3], wk.tail_cap);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < ntask; t += gridDim.x) {
    const TailTask tk = wk.tail[t];
    const QState& S = wk.qs[tk.q];
    const bool on = lane < tk.cnt;
    const int h = wk.surv[(int64_t)tk.q * wk.HCAP + tk.base + (on ? lane : 0)];
#if VL_P32_COPY
    const float* Pq = wk.P32 + (int64_t)tk.q * 12 * wk.HCAP;
    const int col = h;
#else
    const float* Pq = wk.P32s + (int64_t)tk.q * 12 * wk.HCAP;
    const int col = wk.hsrc[(int64_t)tk.q * wk.HCAP + h];
#endif
    float P[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) P[c] = Pq[(int64_t)c * wk.HCAP + col];
    const int NS = S.nsplit, pn = (S.nsub + 1) >> 1, NG = (NS + kGroupSplits - 1) / kGroupSplits;
    const int gfull = S.sA / kGroupSplits, k0 = S.sA % kGroupSplits;
    const float* slot = wk.partial + (int64_t)tk.q * wk.NSPLIT * wk.HCAP + h;  // group g at slot[g * HCAP]
    float c = 0.f, carry = 0.f;
    if (w == 0) {
      for (int g = 0; g < gfull; ++g) c += __ldcg(slot + (int64_t)g * wk.HCAP);
      if (k0) carry = __ldcg(slot + (int64_t)gfull * wk.HCAP);
    }
    const float4* src = wk.sub32 + 3 * (S.sub_off >> 1);
    for (int g = gfull; g < NG; ++g) {
      const int kf = g == gfull ? k0 : 0;  // first split of the group still to score
      const int p0 = g * GP + kf * (kScoreChunk / 2), np = min(GP, pn - g * GP) - kf * (kScoreChunk / 2);
      __syncthreads();  // the previous group's records and split sums are consumed
      for (int k = threadIdx.x; k < 3 * np; k += NT) rec[k] = src[3 * p0 + k];
      __syncthreads();
      const int sp = g * kGroupSplits + w;
      if (w >= kf && sp < NS) {
        float2 acc = make_float2(0.f, 0.f);
        const int pb = (w - kf) * (kScoreChunk / 2), pe = min(pb + kScoreChunk / 2, np);
#pragma unroll 4
        for (int p = pb; p < pe; ++p) {
          const float4 r0 = rec[3 * p], r1 = rec[3 * p + 1], r2 = rec[3 * p + 2];
          const float2 X2 = make_float2(r0.x, r0.y), Y2 = make_float2(r0.z, r0.w);
          const float2 Z2 = make_float2(r1.x, r1.y), A2 = make_float2(r1.z, r1.w);
          const float2 B2 = make_float2(r2.x, r2.y), W2 = make_float2(r2.z, r2.w);
          VL_SCORE_EVAL2(P, acc);
        }
        red[w][lane] = acc.x + acc.y;
      }
      __syncthreads();
      if (w == 0) {
        float gs = kf ? carry : red[0][lane];
        for (int k = kf ? kf : 1; k < kGroupSplits; ++k)
          if (g * kGroupSplits + k < NS) gs += red[k][lane];  // ((p0 + p1) + p2) + p3
        c += gs;
      }
    }
    if (w == 0 && on) wk.cost32[(int64_t)tk.q * wk.HCAP + h] = c;
  }
}

}  // namespace vl
