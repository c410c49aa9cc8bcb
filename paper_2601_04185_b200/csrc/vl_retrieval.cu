// Exact top-K cosine retrieval over the map's global descriptors.
//
// Reference: retrieval.DescriptorIndex.topk (retrieval.py:66-82): sims =
// M @ (q / |q|) in fp64 over unit-normalised rows, order = similarity
// descending, ties by ascending entry id (`rank` = position of the entry id in
// sorted order).  One CTA per query: fp64 dot products (thread per entry for
// short descriptors, warp per entry with a fixed-order butterfly for long
// ones), a register top-K per thread, then K rounds of a block arg-best over
// the per-thread heads.  Deterministic; sims agree with numpy's dgemv to a
// few ulp (summation order), so ids can differ only on near-exact ties.
#include <cfloat>
#include <climits>
#include "vl_common.cuh"

namespace vl {

constexpr int kRetThreads = 256;
constexpr int kRetMaxK = 32;

struct Cand {
  double s;
  int64_t rank;
  int idx;
};

// a precedes b: higher similarity, then lower id rank
__device__ __forceinline__ bool before(const Cand& a, const Cand& b) {
  return a.s > b.s || (a.s == b.s && a.rank < b.rank);
}

__device__ __forceinline__ double norm_inv(const double* q, int D, double* s_red) {
  double acc = 0.0;
  for (int d = threadIdx.x; d < D; d += blockDim.x) acc = fma(q[d], q[d], acc);
  // fixed-order block reduction
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kRetThreads) k_topk(const double* __restrict__ M, const int64_t* __restrict__ rank,
                                                      int E, int D, const double* __restrict__ Qv, int K,
                                                      int* out_idx, double* out_sim, int* bad) {
  __shared__ double s_red[kRetThreads / 32];
  __shared__ double s_q[1024];
  __shared__ Cand s_best[kRetThreads / 32];
  const int qi = blockIdx.x;
  const double* q = Qv + (int64_t)qi * D;
  const double n2 = norm_inv(q, D, s_red);
  const double nrm = sqrt(n2);
  if (!(nrm > 0.0) || !isfinite(nrm)) {
    if (threadIdx.x == 0) atomicOr(bad, 1);
    return;
  }
  const bool smem_q = D <= 1024;
  if (smem_q)
    for (int d = threadIdx.x; d < D; d += kRetThreads) s_q[d] = q[d] / nrm;
  __syncthreads();
  // per-thread sorted top-K (insertion)
  Cand top[kRetMaxK];
  int nt = 0;
  auto push = [&](const Cand& c) {
    if (nt == K && !before(c, top[K - 1])) return;
    int i = nt < K ? nt++ : K - 1;
    while (i > 0 && before(c, top[i - 1])) {
      top[i] = top[i - 1];
      --i;
    }
    top[i] = c;
  };
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (D <= 64) {
    for (int e = threadIdx.x; e < E; e += kRetThreads) {
      const double* r = M + (int64_t)e * D;
      double s = 0.0;
      for (int d = 0; d < D; ++d) s = fma(r[d], smem_q ? s_q[d] : q[d] / nrm, s);
      push(Cand{s, rank[e], e});
    }
  } else {
    // warp per entry: lane-strided partials, fixed butterfly; lane 0 keeps the list
    for (int e = wid; e < E; e += kRetThreads / 32) {
      const double* r = M + (int64_t)e * D;
      double s = 0.0;
      for (int d = lane; d < D; d += 32) s = fma(r[d], smem_q ? s_q[d] : q[d] / nrm, s);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) push(Cand{s, rank[e], e});
    }
  }
  // K rounds of block arg-best over the per-thread heads
  int head = 0;
  for (int k = 0; k < K && k < E; ++k) {
    Cand c = head < nt ? top[head] : Cand{-DBL_MAX, LLONG_MAX, -1};
    for (int o = 16; o > 0; o >>= 1) {
      Cand o_;
      o_.s = __shfl_xor_sync(0xffffffffu, c.s, o);
      o_.rank = __shfl_xor_sync(0xffffffffu, c.rank, o);
      o_.idx = __shfl_xor_sync(0xffffffffu, c.idx, o);
      if (o_.idx >= 0 && (c.idx < 0 || before(o_, c))) c = o_;
    }
    if (lane == 0) s_best[wid] = c;
    __syncthreads();
    Cand b = s_best[0];
    for (int w = 1; w < kRetThreads / 32; ++w)
      if (s_best[w].idx >= 0 && (b.idx < 0 || before(s_best[w], b))) b = s_best[w];
    __syncthreads();
    if (head < nt && top[head].idx == b.idx) ++head;  // the owner pops its head
    if (threadIdx.x == 0) {
      out_idx[(int64_t)qi * K + k] = b.idx;
      out_sim[(int64_t)qi * K + k] = b.s;
    }
  }
}

int launch_topk(const double* M, const int64_t* rank, int E, int D, const double* Qv, int Q, int K, int* out_idx,
                double* out_sim, int* bad, cudaStream_t st) {
  if (Q <= 0) return 0;
  k_topk<<<Q, kRetThreads, 0, st>>>(M, rank, E, D, Qv, K, out_idx, out_sim, bad);
  return 1;
}

}  // namespace vl
