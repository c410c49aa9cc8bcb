// Microbenchmark of k_score2_t variants on synthetic C3-shaped data
// (Q queries x 1530 hypotheses x 10k scoring correspondences).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -I include -I paper_2601_04185_b200/csrc tools/score_bench.cu -o tools/score_bench
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "vl_score.cuh"

using namespace vl;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

struct Bench {
  int Q, nsub, nh, HCAP, NSPLIT;
  Work wk;
  std::vector<QState> hq;
};

template <int NT, int HT, int SPI, int MINB, int UNR>
double run_variant(Bench& b, const char* name, std::vector<float>& ref, int reps, int grid_mult) {
  const int tile = NT * HT;
  const int ntile = (b.nh + tile - 1) / tile;
  const int nsplit = (b.nsub + 127) / 128;
  std::vector<ScoreItem> items;
  for (int q = 0; q < b.Q; ++q)
    for (int t = 0; t < ntile; ++t)
      for (int s = 0; s < nsplit; s += SPI) items.push_back(ScoreItem{q, t, s, nsplit - s < SPI ? nsplit - s : SPI});
  // split count differs per variant: set QState.nsplit accordingly
  for (auto& s : b.hq) s.nsplit = nsplit;
  CK(cudaMemcpy(b.wk.qs, b.hq.data(), b.Q * sizeof(QState), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b.wk.items, items.data(), items.size() * sizeof(ScoreItem), cudaMemcpyHostToDevice));
  int n = (int)items.size();
  CK(cudaMemcpy(b.wk.item_count, &n, sizeof(int), cudaMemcpyHostToDevice));
  int dev = 0, sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int occ = 0;
  auto kern = k_score2_t<NT, HT, SPI, 128, MINB, UNR, false>;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, 0));
  const int grid = sms * occ * grid_mult;
  const float tau2 = 144.f;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t tc_bytes = (size_t)b.Q * b.wk.TCAP * sizeof(int);
  for (int r = 0; r < 2; ++r) {
    cudaMemsetAsync(b.wk.item_count + 1, 0, sizeof(int));
    cudaMemsetAsync(b.wk.tile_cnt, 0, tc_bytes);
    kern<<<grid, NT>>>(b.wk, tau2);
  }
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) {
    cudaMemsetAsync(b.wk.item_count + 1, 0, sizeof(int));
    cudaMemsetAsync(b.wk.tile_cnt, 0, tc_bytes);  // (k_compact does this per round)
    kern<<<grid, NT>>>(b.wk, tau2);
  }
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double evals = (double)b.Q * b.nh * b.nsub * reps;
  const double eps = evals / (ms / 1e3);
  // result: final costs written by the last item of every tile
  std::vector<float> costs((size_t)b.Q * b.HCAP);
  CK(cudaMemcpy(costs.data(), b.wk.cost32, costs.size() * sizeof(float), cudaMemcpyDeviceToHost));
  for (int q = 0; q < b.Q; ++q)
    for (int h = 0; h < b.nh; ++h) costs[(size_t)q * b.nh + h] = costs[(size_t)q * b.HCAP + h];
  costs.resize((size_t)b.Q * b.nh);
  double maxrel = 0;
  if (ref.empty()) ref = costs;
  else
    for (size_t i = 0; i < costs.size(); ++i)
      maxrel = fmax(maxrel, fabs(costs[i] - ref[i]) / fmax(1e-3, fabs(ref[i])));
  printf("%-28s NT=%3d HT=%d SPI=%d minB=%d unr=%d occ=%d grid=%5d  %8.3f ms/rep  %.4e evals/s  %.1f TF(30/eval)  maxrel %.2e\n",
         name, NT, HT, SPI, MINB, UNR, occ, grid, ms / reps, eps, eps * 30 / 1e12, maxrel);
  return eps;
}

int main(int argc, char** argv) {
  Bench b;
  b.Q = argc > 1 ? atoi(argv[1]) : 200;
  b.nsub = 10000;
  b.nh = argc > 3 ? atoi(argv[3]) : 1530;
  b.HCAP = 4000;
  b.NSPLIT = (b.nsub + 127) / 128;
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  // correspondences: points in front of a camera near identity, pixels near projections
  // record pairs (SoA float2 of points 2k, 2k+1: X, Y, Z, cx-u, cy-v, w), the k_prep layout
  std::vector<float4> sub((size_t)b.Q * b.nsub / 2 * 3);
  float* sf = reinterpret_cast<float*>(sub.data());
  for (size_t i = 0; i < (size_t)b.Q * b.nsub; ++i) {
    const float X = 1.2f * U(rng), Y = 1.2f * U(rng), Z = 3.5f + 1.5f * U(rng);
    const float u = 700.f * X / Z + 350.f + 20.f * U(rng), v = 700.f * Y / Z + 350.f + 20.f * U(rng);
    float* pr = sf + 12 * (i >> 1) + (i & 1);
    pr[0] = X, pr[2] = Y, pr[4] = Z, pr[6] = 350.f - u, pr[8] = 350.f - v, pr[10] = 0.5f + 0.5f * fabsf(U(rng));
  }
  std::vector<float> P((size_t)b.Q * 12 * b.HCAP, 0.f);
  for (int q = 0; q < b.Q; ++q)
    for (int h = 0; h < b.nh; ++h) {
      const float a = 0.05f * U(rng), bb = 0.05f * U(rng), tx = 0.1f * U(rng), ty = 0.1f * U(rng);
      const bool garbage = (argc > 2) && (h % 2 == 1);
      const float flip = garbage ? -1.f : 1.f;  // optional: half the hypotheses look backwards
      const float R[9] = {1, -a, bb, a, flip, 0, -bb, 0, flip};
      const float t[3] = {tx, ty, 0.1f * U(rng)};
      float vals[12] = {700 * R[0], 700 * R[1], 700 * R[2], 700 * t[0], 700 * R[3], 700 * R[4],
                        700 * R[5], 700 * t[1], R[6], R[7], R[8], t[2]};
      for (int c = 0; c < 12; ++c) P[((size_t)q * 12 + c) * b.HCAP + h] = vals[c];
    }
  b.hq.resize(b.Q);
  for (int q = 0; q < b.Q; ++q) {
    QState s{};
    s.nh = b.nh;
    s.nsub = b.nsub;
    s.sub_off = (int64_t)q * b.nsub;
    b.hq[q] = s;
  }
  Work& wk = b.wk;
  wk = Work{};
  CK(cudaMalloc(&wk.qs, b.Q * sizeof(QState)));
  CK(cudaMalloc(&wk.sub32, sub.size() * sizeof(float4)));
  CK(cudaMalloc(&wk.P32, P.size() * sizeof(float)));
  CK(cudaMalloc(&wk.partial, (size_t)b.Q * b.NSPLIT * b.HCAP * sizeof(float)));
  CK(cudaMalloc(&wk.items, (size_t)b.Q * 32 * b.NSPLIT * sizeof(ScoreItem)));
  CK(cudaMalloc(&wk.item_count, 2 * sizeof(int)));
  wk.TCAP = (b.HCAP + 255) / 256;
  CK(cudaMalloc(&wk.cost32, (size_t)b.Q * b.HCAP * sizeof(float)));
  CK(cudaMalloc(&wk.tile_cnt, (size_t)b.Q * wk.TCAP * sizeof(int)));
  CK(cudaMemcpy(wk.sub32, sub.data(), sub.size() * sizeof(float4), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(wk.P32, P.data(), P.size() * sizeof(float), cudaMemcpyHostToDevice));
  wk.HCAP = b.HCAP;
  wk.NSPLIT = b.NSPLIT;
  std::vector<float> ref;
  const int reps = 5;
  run_variant<128, 6, 4, 3, 2>(b, "coarse HT6 x4 splits", ref, reps, 1);
  run_variant<128, 2, 1, 6, 2>(b, "fine HT2 x1 split", ref, reps, 1);
  run_variant<128, 4, 4, 4, 2>(b, "HT4 x4 splits", ref, reps, 1);
  return 0;
}
