// Peak-rate probe: scalar FFMA vs packed FFMA2 vs MUFU.RCP mix (tools only).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters, float s) {
  float a[8]; float2 b[8];
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * 1e-3f + j; b[j] = make_float2(a[j], a[j] + 1); }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) a[j] = fmaf(a[j], s, 0.5f);
      if (MODE == 1) b[j] = __ffma2_rn(b[j], make_float2(s, s), make_float2(0.5f, 0.25f));
      if (MODE == 2) { b[j] = __ffma2_rn(b[j], make_float2(s, s), make_float2(0.5f, 0.25f)); a[j] = fmaf(a[j], s, 0.5f); }
    }
  }
  float acc = 0; for (int j = 0; j < 8; ++j) acc += a[j] + b[j].x + b[j].y;
  if (acc == 12345.f) out[0] = acc;
}
int main() {
  float* o; cudaMalloc(&o, 4); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000, grid = sms * 8, block = 256;
  const char* names[3] = {"FFMA", "FFMA2", "FFMA+FFMA2"};
  for (int m = 0; m < 3; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) k<0><<<grid, block>>>(o, iters, 0.999f);
      if (m == 1) k<1><<<grid, block>>>(o, iters, 0.999f);
      if (m == 2) k<2><<<grid, block>>>(o, iters, 0.999f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fma = (double)grid * block * iters * 8 * (m == 0 ? 1 : (m == 1 ? 2 : 3));
      if (rep) printf("%-12s %.2f TFLOP/s\n", names[m], 2 * fma / (ms / 1e3) / 1e12);
    }
  }
}
