// fp32 MSAC hypothesis scoring — kernel template (see vl_score.cu).
#pragma once
#include "vl_internal.h"

namespace vl {

// ---------------------------------------------------------------- f32x2 path
// Blackwell packed FP32 (FFMA2 / FMUL2): one instruction evaluates the same
// step for two hypotheses; the correspondence coordinate is a scalar operand
// broadcast to both halves (SASS `Rn.F32`).  Per pair of evaluations:
// 9 + 1 + 2 + 2 + 1 = 15 FFMA2/FMUL2, 2 MUFU.RSQ, 2 FMNMX — ~10 issue slots
// per evaluation instead of ~17, so the kernel becomes FMA-pipe bound
// rather than issue bound.  Arithmetic per component is identical to the
// scalar path (same fused operations, same order).
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
// only sees the 14 FFMA2/FMUL2 of the evaluation pair.
#define VL_SCORE_EVAL2(Pp, accp)                                                                  \
  {                                                                                               \
    const float2 x_ = fma2(Pp[0], f2(a.x), fma2(Pp[1], f2(a.y), fma2(Pp[2], f2(a.z), Pp[3])));    \
    const float2 y_ = fma2(Pp[4], f2(a.x), fma2(Pp[5], f2(a.y), fma2(Pp[6], f2(a.z), Pp[7])));    \
    const float2 z_ = fma2(Pp[8], f2(a.x), fma2(Pp[9], f2(a.y), fma2(Pp[10], f2(a.z), Pp[11])));  \
    const float2 r_ = make_float2(rcp_approx_ftz(fmaxf(z_.x, 0.f)), rcp_approx_ftz(fmaxf(z_.y, 0.f))); \
    const float2 du_ = fma2(x_, r_, f2(a.w));                                                     \
    const float2 dv_ = fma2(y_, r_, f2(b.x));                                                     \
    float2 e2_ = fma2(du_, du_, mul2(dv_, dv_));                                                  \
    e2_.x = fminf(e2_.x, tau2);                                                                   \
    e2_.y = fminf(e2_.y, tau2);                                                                   \
    accp = fma2(f2(b.y), e2_, accp);                                                              \
  }

// Work item = (query, tile of NT*HT hypotheses, ns <= SPI consecutive
// correspondence splits of SCH records).  The canonical fp32 cost of a
// hypothesis is  sum over split groups (in order) of the group sum
// ((p0 + p1) + p2) + p3  of its splits' sequential record sums — every
// split is accumulated by exactly one thread in record order, so neither the
// tile shape (HT), the splits per item (SPI) nor the grid changes a single
// bit.  The last item to finish a (query, tile) — atomic ticket per tile —
// reduces the tile's partial slots in that order and writes the final costs.
template <int NT, int HT, int SPI, int SCH, int MINB, int UNR>
__global__ void __launch_bounds__(NT, MINB) k_score2_t(Work wk, float tau2) {
  static_assert(HT % 2 == 0, "hypotheses are processed in pairs");
  constexpr int HP = HT / 2;
  constexpr int NW = NT / 32;
  constexpr int WHYP = 32 * HT;  // hypotheses per warp slice
  static_assert(SPI == 1 || SPI == kGroupSplits, "coarse items are exactly one split group");
  __shared__ float4 rec[2 * SPI * SCH];
  __shared__ float red[SPI][SPI > 1 ? NT * HT : 1];
  __shared__ int s_it, s_last;
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
    const int nh = S.nh, nsub = S.nsub;
    const int tile0 = item.tile * (NT * HT);
    const int ns = item.nsplit;
    float* outq = wk.partial + (int64_t)item.q * wk.NSPLIT * wk.HCAP;
    // partial slot layout: fine items (SPI == 1) write one slot per split;
    // coarse items write one slot per group of kGroupSplits splits, holding
    // the group sum ((p0 + p1) + p2) + p3 that k_scan forms itself in fine mode
    const int c0 = item.split * SCH;
    const int cn = min(ns * SCH, nsub - c0);
    const float4* src = wk.sub32 + 2 * (S.sub_off + c0);
    // A partially filled (last) tile of r hypotheses needs WH = ceil(r / WHYP)
    // warp slices; the other warps take other splits of the item (G groups),
    // so a short tile does not leave warps idle.
    const int r = min(NT * HT, nh - tile0);
    const int WH = (r + WHYP - 1) / WHYP;
    const int G = NW / WH;
    const int hs = w % WH, grp = w / WH;
    __syncthreads();
    for (int k = threadIdx.x; k < 2 * cn; k += NT) rec[k] = src[k];
    float2 P[HP][12];
    int hid[HT];
    const float* Pq = wk.P32 + (int64_t)item.q * 12 * wk.HCAP;
#pragma unroll
    for (int j = 0; j < HT; ++j) hid[j] = tile0 + hs * WHYP + lane * HT + j;
#pragma unroll
    for (int jp = 0; jp < HP; ++jp) {
      const int h0 = hid[2 * jp] < nh ? hid[2 * jp] : 0;
      const int h1 = hid[2 * jp + 1] < nh ? hid[2 * jp + 1] : 0;
#pragma unroll
      for (int c = 0; c < 12; ++c)
        P[jp][c] = make_float2(Pq[(int64_t)c * wk.HCAP + h0], Pq[(int64_t)c * wk.HCAP + h1]);
    }
    __syncthreads();
    float2 gsum[HP];
#pragma unroll
    for (int jp = 0; jp < HP; ++jp) gsum[jp] = make_float2(0.f, 0.f);
    for (int s = grp; s < ns && grp < G; s += G) {
      float2 acc[HP];
#pragma unroll
      for (int jp = 0; jp < HP; ++jp) acc[jp] = make_float2(0.f, 0.f);
      const int cb = s * SCH, ce = min(cb + SCH, cn);
#pragma unroll UNR
      for (int c = cb; c < ce; ++c) {
        const float4 a = rec[2 * c];
        const float4 b = rec[2 * c + 1];
#pragma unroll
        for (int jp = 0; jp < HP; ++jp) VL_SCORE_EVAL2(P[jp], acc[jp]);
      }
      if (SPI == 1) {
        float* out = outq + (int64_t)(item.split + s) * wk.HCAP;
#pragma unroll
        for (int jp = 0; jp < HP; ++jp) {
          if (hid[2 * jp] < nh) out[hid[2 * jp]] = acc[jp].x;
          if (hid[2 * jp + 1] < nh) out[hid[2 * jp + 1]] = acc[jp].y;
        }
      } else if (G == 1) {
#pragma unroll
        for (int jp = 0; jp < HP; ++jp) {
          gsum[jp].x = (s == 0) ? acc[jp].x : gsum[jp].x + acc[jp].x;
          gsum[jp].y = (s == 0) ? acc[jp].y : gsum[jp].y + acc[jp].y;
        }
      } else {
        // split s of a partial tile computed by warp group grp: park it
#pragma unroll
        for (int jp = 0; jp < HP; ++jp) {
          red[s][hs * WHYP + lane * HT + 2 * jp] = acc[jp].x;
          red[s][hs * WHYP + lane * HT + 2 * jp + 1] = acc[jp].y;
        }
      }
    }
    if (SPI > 1) {
      float* out = outq + (int64_t)(item.split / kGroupSplits) * wk.HCAP;
      if (G > 1) {
        __syncthreads();
        if (grp == 0) {
#pragma unroll
          for (int jp = 0; jp < HP; ++jp) {
            float sx = red[0][hs * WHYP + lane * HT + 2 * jp], sy = red[0][hs * WHYP + lane * HT + 2 * jp + 1];
            for (int s = 1; s < ns; ++s) {
              sx += red[s][hs * WHYP + lane * HT + 2 * jp];
              sy += red[s][hs * WHYP + lane * HT + 2 * jp + 1];
            }
            gsum[jp] = make_float2(sx, sy);
          }
        }
      }
      if (grp == 0) {
#pragma unroll
        for (int jp = 0; jp < HP; ++jp) {
          if (hid[2 * jp] < nh) out[hid[2 * jp]] = gsum[jp].x;
          if (hid[2 * jp + 1] < nh) out[hid[2 * jp + 1]] = gsum[jp].y;
        }
      }
    }
    // ---- tile completion ticket (threadfence reduction pattern)
    __threadfence();
    __syncthreads();
    const int NS = S.nsplit;
    const int NG = (NS + kGroupSplits - 1) / kGroupSplits;
    if (threadIdx.x == 0) {
      const int tile_items = SPI == 1 ? NS : NG;
      s_last = atomicAdd(wk.tile_cnt + (int64_t)item.q * wk.TCAP + item.tile, 1) == tile_items - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      const int h1 = min(nh, tile0 + NT * HT);
      float* costq = wk.cost32 + (int64_t)item.q * wk.HCAP;
      for (int h = tile0 + threadIdx.x; h < h1; h += NT) {
        float c = 0.f;
        if (SPI == 1) {
          for (int g = 0; g < NG; ++g) {
            float v[kGroupSplits];
#pragma unroll
            for (int k = 0; k < kGroupSplits; ++k) {
              const int sp = g * kGroupSplits + k;
              v[k] = sp < NS ? __ldcg(outq + (int64_t)sp * wk.HCAP + h) : 0.f;
            }
            float gs = v[0];
#pragma unroll
            for (int k = 1; k < kGroupSplits; ++k)
              if (g * kGroupSplits + k < NS) gs += v[k];
            c += gs;
          }
        } else {
          int g = 0;
          for (; g + 4 <= NG; g += 4) {
            float v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = __ldcg(outq + (int64_t)(g + k) * wk.HCAP + h);
#pragma unroll
            for (int k = 0; k < 4; ++k) c += v[k];
          }
          for (; g < NG; ++g) c += __ldcg(outq + (int64_t)g * wk.HCAP + h);
        }
        costq[h] = c;
      }
    }
  }
}

}  // namespace vl
