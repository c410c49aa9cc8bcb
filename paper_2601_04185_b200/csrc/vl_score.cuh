// fp32 MSAC hypothesis scoring — kernel template (see vl_score.cu).
#pragma once
#include "vl_internal.h"

namespace vl {

__device__ __forceinline__ float rsqrt_approx_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// One evaluation: e = w * min(|pi(P X) - px|^2, tau^2), behind-camera -> tau^2.
// P rows are pre-multiplied by fx / fy; a.w, b.x hold f32(cx - u), f32(cy - v).
#define VL_SCORE_EVAL(Pj, accj)                                                       \
  {                                                                                   \
    const float x_ = fmaf(Pj[0], a.x, fmaf(Pj[1], a.y, fmaf(Pj[2], a.z, Pj[3])));     \
    const float y_ = fmaf(Pj[4], a.x, fmaf(Pj[5], a.y, fmaf(Pj[6], a.z, Pj[7])));     \
    const float z_ = fmaf(Pj[8], a.x, fmaf(Pj[9], a.y, fmaf(Pj[10], a.z, Pj[11])));   \
    const float rs_ = rsqrt_approx_ftz(z_);                                           \
    const float r_ = rs_ * rs_;                                                       \
    const float du_ = fmaf(x_, r_, a.w);                                              \
    const float dv_ = fmaf(y_, r_, b.x);                                              \
    const float e2_ = fminf(fmaf(du_, du_, dv_ * dv_), tau2);                         \
    accj = fmaf(b.y, e2_, accj);                                                      \
  }

// Persistent grid over work items (query, tile of NT*HT hypotheses, split of
// CH correspondences).  Thread t owns hypotheses tile*NT*HT + j*NT + t.
template <int NT, int HT, int CH, int MINB, int UNR>
__global__ void __launch_bounds__(NT, MINB) k_score_t(Work wk, float tau2) {
  __shared__ float4 rec[2 * CH];
  const int nitems = *wk.item_count;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const ScoreItem item = wk.items[it];
    const QState& S = wk.qs[item.q];
    const int nh = S.nh, nsub = S.nsub;
    const int c0 = item.split * CH;
    const int cn = min(CH, nsub - c0);
    const float4* src = wk.sub32 + 2 * (S.sub_off + c0);
    __syncthreads();
    for (int k = threadIdx.x; k < 2 * cn; k += NT) rec[k] = src[k];
    float P[HT][12];
    int hid[HT];
    const float* Pq = wk.P32 + (int64_t)item.q * 12 * wk.HCAP;
#pragma unroll
    for (int j = 0; j < HT; ++j) {
      const int h = item.tile * (NT * HT) + j * NT + threadIdx.x;
      hid[j] = h;
      const int hc = h < nh ? h : 0;
#pragma unroll
      for (int c = 0; c < 12; ++c) P[j][c] = Pq[(int64_t)c * wk.HCAP + hc];
    }
    __syncthreads();
    float acc[HT];
#pragma unroll
    for (int j = 0; j < HT; ++j) acc[j] = 0.f;
#pragma unroll UNR
    for (int c = 0; c < cn; ++c) {
      const float4 a = rec[2 * c];
      const float4 b = rec[2 * c + 1];
#pragma unroll
      for (int j = 0; j < HT; ++j) VL_SCORE_EVAL(P[j], acc[j]);
    }
    float* out = wk.partial + ((int64_t)item.q * wk.NSPLIT + item.split) * wk.HCAP;
#pragma unroll
    for (int j = 0; j < HT; ++j)
      if (hid[j] < nh) out[hid[j]] = acc[j];
  }
}

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
// hypothesis is  sum over splits (in order) of  [sequential sum over the
// split's records]  — every split is accumulated by exactly one thread in
// record order and written to its own partial slot, so neither the tile
// shape (HT), the splits per item (SPI) nor the grid changes a single bit.
template <int NT, int HT, int SPI, int SCH, int MINB, int UNR>
__global__ void __launch_bounds__(NT, MINB) k_score2_t(Work wk, float tau2) {
  static_assert(HT % 2 == 0, "hypotheses are processed in pairs");
  constexpr int HP = HT / 2;
  constexpr int NW = NT / 32;
  constexpr int WHYP = 32 * HT;  // hypotheses per warp slice
  static_assert(SPI == 1 || SPI == kGroupSplits, "coarse items are exactly one split group");
  __shared__ float4 rec[2 * SPI * SCH];
  __shared__ float red[SPI][SPI > 1 ? NT * HT : 1];
  __shared__ int s_it;
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
    if (wk.split_size > 1 && it % wk.split_size != wk.split_rank) {
      // hypothesis-split mode: another rank owns this item; contribute zeros
      // to the SUM all-reduce of the partial buffer
      const int h1 = min(nh, tile0 + NT * HT);
      const int slot0 = SPI == 1 ? item.split : item.split / kGroupSplits;
      const int nslot = SPI == 1 ? ns : 1;
      for (int s = 0; s < nslot; ++s)
        for (int h = tile0 + threadIdx.x; h < h1; h += NT) outq[(int64_t)(slot0 + s) * wk.HCAP + h] = 0.f;
      __syncthreads();  // every thread has read s_it before it is rewritten
      continue;
    }
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
  }
}

}  // namespace vl
