/*
 * Plain-C client of the C ABI (include/visloc_b200.h): no Python, no torch.
 *
 *   gcc -O2 -std=c11 tools/capi_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2601_04185_b200/_lib -L/usr/local/cuda/lib64 -lvisloc_b200 -lcudart \
 *       -Wl,-rpath,paper_2601_04185_b200/_lib -o /tmp/capi_demo && /tmp/capi_demo
 *
 * Builds Q synthetic queries (the generator-A model of test_posest.py:22-35:
 * camera-frame points, a ground-truth pose, 30 % inliers with 1 px noise,
 * uniform outliers), estimates them with one vl_ransac_pnp call (device
 * arrays from cudaMalloc, per-query numpy-seeded PCG64 states from
 * vl_pcg64_seed), checks every pose against the ground truth, scores the
 * ground truth with vl_msac_score and exercises the error paths (n < 3,
 * bad config).  Prints one summary line; exit status 0 on success.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "visloc_b200.h"

#define CHECK(x)                                                                 \
  do {                                                                           \
    int rc_ = (x);                                                               \
    if (rc_ != VL_OK) {                                                          \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, vl_last_error(ctx));      \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

static uint64_t rs = 0x9E3779B97F4A7C15ull;
static double urand(void) { /* xorshift64*, uniform [0, 1) */
  rs ^= rs >> 12;
  rs ^= rs << 25;
  rs ^= rs >> 27;
  return (double)((rs * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0);
}
static double nrand(void) {
  const double u = urand() + 1e-300, v = urand();
  return sqrt(-2.0 * log(u)) * cos(6.283185307179586 * v);
}

/* rotation matrix of a unit quaternion (w, x, y, z) */
static void q2R(const double* q, double* R) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

int main(int argc, char** argv) {
  const int Q = argc > 1 ? atoi(argv[1]) : 64, n = 5000;
  const double fx = 700, fy = 700, cx = 350, cy = 350;
  vl_ctx* ctx = NULL;
  if (vl_create(0, &ctx) != VL_OK) {
    fprintf(stderr, "vl_create failed (a B200 / sm_100 GPU is required)\n");
    return 1;
  }
  double *px = malloc(sizeof(double) * 2 * n * Q), *X = malloc(sizeof(double) * 3 * n * Q),
         *w = malloc(sizeof(double) * n * Q), *gq = malloc(sizeof(double) * 4 * Q), *gt = malloc(sizeof(double) * 3 * Q);
  int64_t* offsets = malloc(sizeof(int64_t) * (Q + 1));
  vl_intrinsics* intr = malloc(sizeof(vl_intrinsics) * Q);
  vl_pcg64_state* rng = malloc(sizeof(vl_pcg64_state) * Q);
  for (int q = 0; q < Q; ++q) {
    double qq[4] = {1.0, 0.05 * nrand(), 0.05 * nrand(), 0.05 * nrand()}, R[9];
    const double nq = sqrt(qq[0] * qq[0] + qq[1] * qq[1] + qq[2] * qq[2] + qq[3] * qq[3]);
    for (int k = 0; k < 4; ++k) gq[4 * q + k] = qq[k] / nq;
    q2R(gq + 4 * q, R);
    for (int k = 0; k < 3; ++k) gt[3 * q + k] = 0.2 * nrand();
    for (int i = 0; i < n; ++i) {
      const int64_t r = (int64_t)q * n + i;
      const double xc[3] = {2.4 * urand() - 1.2, 2.4 * urand() - 1.2, 2.0 + 3.0 * urand()};
      /* world point X = R^T (xc - t) */
      for (int a = 0; a < 3; ++a) {
        double s = 0;
        for (int b = 0; b < 3; ++b) s += R[3 * b + a] * (xc[b] - gt[3 * q + b]);
        X[3 * r + a] = s;
      }
      if (urand() < 0.3) {  /* inlier */
        px[2 * r] = fx * xc[0] / xc[2] + cx + nrand();
        px[2 * r + 1] = fy * xc[1] / xc[2] + cy + nrand();
        w[r] = 0.5 + 0.5 * urand();
      } else {
        px[2 * r] = 700 * urand();
        px[2 * r + 1] = 700 * urand();
        w[r] = 0.05 + 0.25 * urand();
      }
    }
    offsets[q] = (int64_t)q * n;
    intr[q] = (vl_intrinsics){fx, fy, cx, cy};
    CHECK(vl_pcg64_seed((uint64_t)(1000 + q), &rng[q]));  /* == np.random.default_rng(1000 + q) */
  }
  offsets[Q] = (int64_t)Q * n;
  const size_t N = (size_t)n * Q;
  double *dpx, *dX, *dw, *dq, *dt, *dscore;
  uint8_t* dflags;
  int64_t *dcnt, *dit, *dstats;
  int32_t* dconv;
  if (cudaMalloc((void**)&dpx, 16 * N) || cudaMalloc((void**)&dX, 24 * N) || cudaMalloc((void**)&dw, 8 * N) ||
      cudaMalloc((void**)&dq, 32 * Q) || cudaMalloc((void**)&dt, 24 * Q) || cudaMalloc((void**)&dscore, 8 * Q) ||
      cudaMalloc((void**)&dflags, N) || cudaMalloc((void**)&dcnt, 8 * Q) || cudaMalloc((void**)&dit, 8 * Q) ||
      cudaMalloc((void**)&dstats, 32 * Q) || cudaMalloc((void**)&dconv, 4 * Q)) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  cudaMemcpy(dpx, px, 16 * N, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X, 24 * N, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, w, 8 * N, cudaMemcpyHostToDevice);

  vl_ransac_args args;
  memset(&args, 0, sizeof args);
  args.num_queries = Q;
  args.offsets = offsets;
  args.intr = intr;
  args.rng = rng;
  args.px = dpx;
  args.X = dX;
  args.w = dw;
  args.cfg.max_iterations = 100000;  /* RansacConfig() defaults (posest.py:69-90) */
  args.cfg.batch_size = 1000;
  args.cfg.max_scoring = 10000;
  args.cfg.miss_probability = 1e-4;
  args.cfg.reproj_threshold = 12.0;
  args.cfg.cauchy_scale = 0.0;  /* None -> tau */
  args.cfg.lm_max_iters = 100;
  vl_ransac_out out = {dq, dt, dflags, dcnt, dscore, dit, dconv, dstats};
  CHECK(vl_ransac_pnp(ctx, &args, &out, NULL));
  CHECK(cudaDeviceSynchronize() == cudaSuccess ? VL_OK : VL_ERR_CUDA);

  double* hq = malloc(32 * Q);
  double* ht = malloc(24 * Q);
  int32_t* hconv = malloc(4 * Q);
  int64_t* hcnt = malloc(8 * Q);
  cudaMemcpy(hq, dq, 32 * Q, cudaMemcpyDeviceToHost);
  cudaMemcpy(ht, dt, 24 * Q, cudaMemcpyDeviceToHost);
  cudaMemcpy(hconv, dconv, 4 * Q, cudaMemcpyDeviceToHost);
  cudaMemcpy(hcnt, dcnt, 8 * Q, cudaMemcpyDeviceToHost);
  double worst_deg = 0, worst_t = 0;
  int conv = 0;
  for (int q = 0; q < Q; ++q) {
    double d = fabs(hq[4 * q] * gq[4 * q] + hq[4 * q + 1] * gq[4 * q + 1] + hq[4 * q + 2] * gq[4 * q + 2] +
                    hq[4 * q + 3] * gq[4 * q + 3]);
    if (d > 1) d = 1;
    const double deg = 2 * acos(d) * 57.29577951308232;
    double et = 0;
    for (int k = 0; k < 3; ++k) et += (ht[3 * q + k] - gt[3 * q + k]) * (ht[3 * q + k] - gt[3 * q + k]);
    if (deg > worst_deg) worst_deg = deg;
    if (sqrt(et) > worst_t) worst_t = sqrt(et);
    conv += hconv[q] ? 1 : 0;
  }
  /* MSAC cost of the ground truth of query 0 (posest.msac_score) */
  double gt_cost = 0;
  CHECK(vl_msac_score(ctx, gq, gt, dpx, dX, dw, n, intr[0], 12.0, &gt_cost, NULL, NULL));
  /* error paths: n < 3 -> VL_ERR_UNDERCONSTRAINED, tau <= 0 -> VL_ERR_INVALID */
  int64_t off2[2] = {0, 2};
  vl_ransac_args bad = args;
  bad.num_queries = 1;
  bad.offsets = off2;
  const int e1 = vl_ransac_pnp(ctx, &bad, &out, NULL);
  bad = args;
  bad.cfg.reproj_threshold = -1;
  const int e2 = vl_ransac_pnp(ctx, &bad, &out, NULL);
  printf("capi_demo: queries %d converged %d worst rotation %.2e deg worst |dt| %.2e inliers[0] %lld "
         "gt msac cost %.1f err_codes %d %d launches %lld\n",
         Q, conv, worst_deg, worst_t, (long long)hcnt[0], gt_cost, e1, e2, (long long)vl_launch_count(ctx));
  vl_destroy(ctx);
  const int ok = conv == Q && worst_deg < 0.2 && worst_t < 0.02 && e1 == VL_ERR_UNDERCONSTRAINED &&
                 e2 == VL_ERR_INVALID && gt_cost > 0;
  return ok ? 0 : 2;
}
