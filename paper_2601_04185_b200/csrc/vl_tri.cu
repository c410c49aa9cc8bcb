// Dense per-pixel depth triangulation against covisible posed views.
//
// Reference: depthbuild.build_depth_map (depthbuild.py:249-375) with
// _vec_cost / _vec_gradient / _refine_depth_vec (:378-441), and the scalar
// path triangulate_pixel / depth_hypothesis / _refine_depth_scalar
// (:104-227) for explicit observation sets.
//
// Layout: a GROUP of G lanes (8, 16 or 32) owns one pixel; lane l holds the
// pixel's observations v = s*G + l (s < OPL slots), i.e. the views of the
// covisible set.  Per pixel:
//   1. observation setup (gate, world bearing, closest-point depth
//      hypothesis), one view per lane;
//   2. voting: every hypothesis j (broadcast by shuffle) is tested against
//      the lane's observations; the inlier count is a group ballot popcount
//      and the winner is the first maximum (strict >), its inlier ballots kept;
//   3. damped Newton on the confidence-weighted squared angular error over
//      the winner's inlier set.  Every sum over views is gathered by shuffles
//      in view order and added with numpy's pairwise-summation scheme (8
//      rotating partial sums), so all lanes hold bit-identical sums and the
//      control flow of the line search is group-uniform.
// Element-wise arithmetic follows the reference's operation order
// (numpy matmul = FMA chain, einsum = (a0b0 + a2b2) + a1b1, np.sum over 3 =
// sequential, no FMA contraction elsewhere); arctan2 is CUDA's (a few ulp
// from glibc), so depths agree with the reference to ~1e-15 relative and
// round to the same f32 almost always.
//
// Voting avoids the arctan2: for thr < pi/2, atan2(s, c) < thr <=> c > 0 and
// s^2 < c^2 tan^2(thr); the comparison is decided from squares when it is
// not within 1e-10 relative of the boundary, otherwise by the reference's
// exact expression atan2(sqrt(s^2), c) < thr.
//
// Bound: fp64 latency/ALU (V^2 vote tests + ~10 V-term sums per Newton step
// per pixel); inputs are 12-24 B per (pixel, view).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>
#include "vl_common.cuh"

namespace vl {

struct TriView {  // vl_tri_view
  const void* targets;
  const void* confidence;
  double rt[9];
  double center[3];
  double fx, fy, cx, cy;
};
struct TriMap {  // vl_tri_map
  int32_t grid_w, grid_h, view0, nview;
  double fx, fy, cx, cy;
  double sx, sy;
  double R[9];
  double center[3];
  float* depth;
  uint8_t* valid;
};
struct TriConfig {  // vl_tri_config
  double thr, conf_thr, refine_tol;
  int32_t min_inliers, max_refine_iters;
};
struct TriProblem {  // vl_tri_problem
  double ray[3], center[3];
  int32_t obs0, nobs;
};
struct TriObs {  // vl_tri_obs
  double rt[9], center[3];
  double fx, fy, cx, cy;
  double target[2];
  double confidence;
};

static_assert(sizeof(TriView) == 144 && sizeof(TriMap) == 176 && sizeof(TriProblem) == 56 &&
                  sizeof(TriObs) == 152 && sizeof(TriConfig) == 32, "C ABI layouts (visloc_b200.h)");

constexpr int kTriThreads = 128;
#ifndef VL_TRI_MINB
#define VL_TRI_MINB 1  // min resident CTAs per SM for the map kernel (register cap)
#endif
constexpr double kParallelTol = 1e-12;  // depthbuild.py:42

VL_HD double ddiv(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}

// numpy pairwise_sum (n <= 128): 8 partial sums over the first n - n%8
// terms, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the rest added
// sequentially.  Terms arrive in order; the partials rotate so element i
// always lands in partial i%8 without dynamic register indexing.
struct PwSum {
  double r0, r1, r2, r3, r4, r5, r6, r7, res;
  int i, tail;
  __device__ __forceinline__ void init(int n) {
    r0 = r1 = r2 = r3 = r4 = r5 = r6 = r7 = 0.0;
    res = 0.0;
    i = 0;
    tail = n < 8 ? 0 : n - (n & 7);
  }
  __device__ __forceinline__ double combine() const {
    return dadd(dadd(dadd(r0, r1), dadd(r2, r3)), dadd(dadd(r4, r5), dadd(r6, r7)));
  }
  __device__ __forceinline__ void add(double x) {
    if (i < tail) {
      const double t = dadd(r0, x);
      r0 = r1; r1 = r2; r2 = r3; r3 = r4; r4 = r5; r5 = r6; r6 = r7; r7 = t;
    } else {
      if (i == tail) res = tail ? combine() : 0.0;
      res = dadd(res, x);
    }
    ++i;
  }
  __device__ __forceinline__ double get() const {
    if (i <= tail) return tail ? combine() : 0.0;
    return res;
  }
};

// Per-lane observations of one pixel (slot s holds view s*G + lane).
template <int OPL>
struct LaneObs {
  double b[OPL][3];   // world bearing (0 where gated out)
  double c[OPL][3];   // view centre
  double conf[OPL];
  double D[OPL];      // depth hypothesis along the reference ray
  bool ok[OPL], hok[OPL];
};

__device__ __forceinline__ void cross3(const double* a, const double* b, double* o) {
  o[0] = dsub(dmul(a[1], b[2]), dmul(a[2], b[1]));
  o[1] = dsub(dmul(a[2], b[0]), dmul(a[0], b[2]));
  o[2] = dsub(dmul(a[0], b[1]), dmul(a[1], b[0]));
}
__device__ __forceinline__ double sum3(double a, double b, double c) { return dadd(dadd(a, b), c); }
__device__ __forceinline__ double dot3(const double* a, const double* b) {  // np.sum(a*b, axis=-1)
  return sum3(dmul(a[0], b[0]), dmul(a[1], b[1]), dmul(a[2], b[2]));
}
__device__ __forceinline__ double einsum3(const double* a, const double* b) {  // einsum "...d,...d"
  return dadd(dadd(dmul(a[0], b[0]), dmul(a[2], b[2])), dmul(a[1], b[1]));
}
__device__ __forceinline__ double matmul3(const double* a, const double* b) {  // BLAS dot: FMA chain
  return fma(a[2], b[2], fma(a[1], b[1], dmul(a[0], b[0])));
}

// world bearing of a target pixel seen by a view (depthbuild.py:302-310)
__device__ __forceinline__ void view_bearing(const double* rt, double fx, double fy, double cx, double cy, double tx,
                                             double ty, double* b) {
  const double bx = ddiv(dsub(tx, cx), fx), by = ddiv(dsub(ty, cy), fy);
  const double n = sqrt(sum3(dmul(bx, bx), dmul(by, by), 1.0));
  const double bc[3] = {ddiv(bx, n), ddiv(by, n), ddiv(1.0, n)};
#pragma unroll
  for (int i = 0; i < 3; ++i) b[i] = einsum3(rt + 3 * i, bc);
}

// closest point on the reference ray (depthbuild.py:322-328)
__device__ __forceinline__ void hypothesis(const double* ray, const double* cref, const double* b, const double* cv,
                                           bool ok, double& D, bool& hok) {
  const double w[3] = {dsub(cv[0], cref[0]), dsub(cv[1], cref[1]), dsub(cv[2], cref[2])};
  const double A = matmul3(ray, w);
  const double beta = einsum3(b, ray);
  const double Bw = einsum3(b, w);
  const double denom = dsub(1.0, dmul(beta, beta));
  D = ddiv(dsub(A, dmul(beta, Bw)), denom);
  hok = ok && denom >= kParallelTol && isfinite(D) && D > 0.0;
}

// angle(pred, b) < thr (depthbuild.py:344-348), exact near the boundary
__device__ __forceinline__ bool angle_below(const double* pred, const double* b, double thr, double tan2, bool fast) {
  double cr[3];
  cross3(pred, b, cr);
  const double s2 = sum3(dmul(cr[0], cr[0]), dmul(cr[1], cr[1]), dmul(cr[2], cr[2]));
  const double c = dot3(pred, b);
  if (fast) {
    if (!(c > 0.0)) return false;
    const double rhs = c * c * tan2;
    const double diff = s2 - rhs;
    if (fabs(diff) > 1e-10 * (s2 + rhs)) return diff < 0.0;
  }
  return atan2(sqrt(s2), c) < thr;
}

__device__ __forceinline__ void point_on_ray(const double* cref, double d, const double* ray, double* X) {
#pragma unroll
  for (int i = 0; i < 3; ++i) X[i] = dadd(cref[i], dmul(d, ray[i]));
}

// Sum over the pixel's views of per-lane terms, in numpy's pairwise order,
// identical in every lane of the group.  vec mode (all V positions, zeros
// off the inlier set): the 8 partial sums r_j = x_j + x_{j+8} + ... are
// gathered by lanes j (mod 8) with one shuffle per 8 elements, combined by a
// 3-level xor butterfly (== ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), addition
// being commutative) and the n%8 tail is added in order.  scalar mode (the
// inlier subset only, triangulate_pixel): serial gather through PwSum.
template <int G, int OPL>
__device__ __forceinline__ double group_sum(const double* term, const uint32_t* inl, int V, int nin, int lane,
                                            unsigned gmask, bool scalar_mode) {
  if (scalar_mode) {
    PwSum acc;
    acc.init(nin);
#pragma unroll
    for (int s = 0; s < OPL; ++s)
      for (int l = 0; l < G; ++l) {
        const int v = s * G + l;
        if (v >= V) break;
        const double x = __shfl_sync(gmask, term[s], l, G);
        if ((inl[s] >> l) & 1u) acc.add(x);
      }
    return acc.get();
  }
  const int n = V;
  if (n < 8) {  // sequential from 0 (all in slot 0: G >= 8)
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = dadd(res, __shfl_sync(gmask, term[0], i, G));
    return res;
  }
  const int tail = n - (n & 7);
  double r = 0.0;
#pragma unroll
  for (int s = 0; s < OPL; ++s)
#pragma unroll
    for (int b = 0; b < G; b += 8) {
      const int base = s * G + b;  // elements base .. base+7
      if (base < tail) {
        const double v = __shfl_sync(gmask, term[s], b + (lane & 7), G);
        r = base == 0 ? v : dadd(r, v);
      }
    }
  r = dadd(r, __shfl_xor_sync(gmask, r, 1, G));
  r = dadd(r, __shfl_xor_sync(gmask, r, 2, G));
  r = dadd(r, __shfl_xor_sync(gmask, r, 4, G));
#pragma unroll
  for (int s = 0; s < OPL; ++s)
    for (int l = 0; l < G; ++l) {
      const int i = s * G + l;
      if (i >= n) break;
      if (i >= tail) r = dadd(r, __shfl_sync(gmask, term[s], l, G));
    }
  return r;
}

// Weighted squared angular error (scalar_mode: sum over the inlier subset only)
template <int G, int OPL>
__device__ double tri_cost(const LaneObs<OPL>& o, const uint32_t* inl, int V, int nin, double d, const double* ray,
                           const double* cref, int lane, unsigned gmask, bool scalar_mode) {
  double X[3];
  point_on_ray(cref, d, ray, X);
  double term[OPL];
#pragma unroll
  for (int s = 0; s < OPL; ++s) {
    term[s] = 0.0;
    if ((inl[s] >> lane) & 1u) {
      const double pred[3] = {dsub(X[0], o.c[s][0]), dsub(X[1], o.c[s][1]), dsub(X[2], o.c[s][2])};
      double cr[3];
      cross3(pred, o.b[s], cr);
      const double ang = atan2(sqrt(sum3(dmul(cr[0], cr[0]), dmul(cr[1], cr[1]), dmul(cr[2], cr[2]))),
                               dot3(pred, o.b[s]));
      term[s] = dmul(dmul(o.conf[s], ang), ang);
    }
  }
  return group_sum<G, OPL>(term, inl, V, nin, lane, gmask, scalar_mode);
}

template <int G, int OPL>
__device__ double tri_grad(const LaneObs<OPL>& o, const uint32_t* inl, int V, int nin, double d, const double* ray,
                           const double* cref, int lane, unsigned gmask, bool scalar_mode) {
  double X[3];
  point_on_ray(cref, d, ray, X);
  double term[OPL];
#pragma unroll
  for (int s = 0; s < OPL; ++s) {
    term[s] = 0.0;
    if ((inl[s] >> lane) & 1u) {
      const double* b = o.b[s];
      const double pred[3] = {dsub(X[0], o.c[s][0]), dsub(X[1], o.c[s][1]), dsub(X[2], o.c[s][2])};
      double cr[3], rb[3];
      cross3(pred, b, cr);
      const double sn = sqrt(sum3(dmul(cr[0], cr[0]), dmul(cr[1], cr[1]), dmul(cr[2], cr[2])));
      const double c = dot3(pred, b);
      const double theta = atan2(sn, c);
      cross3(ray, b, rb);
      double s_p, th_p;
      if (scalar_mode) {  // depthbuild.py:195-198
        s_p = sn > 1e-300 ? ddiv(dot3(cr, rb), sn > 0.0 ? sn : 1.0) : 0.0;
        const double c_p = matmul3(b, ray);
        th_p = ddiv(dsub(dmul(s_p, c), dmul(sn, c_p)), dadd(dmul(sn, sn), dmul(c, c)));
      } else {  // depthbuild.py:395-402
        s_p = sn > 0.0 ? ddiv(dot3(cr, rb), sn) : 0.0;
        const double c_p = dot3(b, ray);
        const double n2 = dadd(dmul(sn, sn), dmul(c, c));
        th_p = n2 > 0.0 ? ddiv(dsub(dmul(s_p, c), dmul(sn, c_p)), n2) : 0.0;
      }
      term[s] = dmul(dmul(dmul(2.0, o.conf[s]), theta), th_p);
    }
  }
  return group_sum<G, OPL>(term, inl, V, nin, lane, gmask, scalar_mode);
}

// Voting + refinement of one pixel; returns the winner's inlier count (0 if
// no hypothesis reaches min_inliers) and the refined ray depth.
template <int G, int OPL>
__device__ int tri_solve(const LaneObs<OPL>& o, int V, const double* ray, const double* cref, const TriConfig& cfg,
                         int lane, unsigned gmask, int gbase, bool scalar_mode, double& d_out) {
  const double tan_t = tan(cfg.thr);
  const bool fast = cfg.thr > 0.0 && cfg.thr < 1.5;
  const double tan2 = tan_t * tan_t;
  int best = 0;
  uint32_t best_inl[OPL];
  double best_d = 0.0;
#pragma unroll
  for (int s = 0; s < OPL; ++s) best_inl[s] = 0u;
#pragma unroll
  for (int sj = 0; sj < OPL; ++sj)
    for (int lj = 0; lj < G; ++lj) {
      const int j = sj * G + lj;
      if (j >= V) break;
      const double Dj = __shfl_sync(gmask, o.D[sj], lj, G);
      const bool hj = __shfl_sync(gmask, (int)o.hok[sj], lj, G);
      if (!hj) continue;
      double X[3];
      point_on_ray(cref, Dj, ray, X);
      int count = 0;
      uint32_t m[OPL];
#pragma unroll
      for (int s = 0; s < OPL; ++s) {
        bool in = false;
        if (o.ok[s]) {
          const double pred[3] = {dsub(X[0], o.c[s][0]), dsub(X[1], o.c[s][1]), dsub(X[2], o.c[s][2])};
          in = angle_below(pred, o.b[s], cfg.thr, tan2, fast);
        }
        m[s] = (__ballot_sync(gmask, in) >> gbase) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u));
        count += __popc(m[s]);
      }
      if (count > best) {  // strict: the first maximum wins (np.argmax)
        best = count;
        best_d = Dj;
#pragma unroll
        for (int s = 0; s < OPL; ++s) best_inl[s] = m[s];
      }
    }
  if (best < cfg.min_inliers || best == 0) return 0;
  // damped Newton (depthbuild.py:408-441 / :208-227)
  const int nin = best;
  double d = best_d;
  double cost = tri_cost<G, OPL>(o, best_inl, V, nin, d, ray, cref, lane, gmask, scalar_mode);
  for (int it = 0; it < cfg.max_refine_iters; ++it) {
    const double g = tri_grad<G, OPL>(o, best_inl, V, nin, d, ray, cref, lane, gmask, scalar_mode);
    const double h = fmax(dmul(1e-7, fabs(d)), 1e-10);
    const double gp = tri_grad<G, OPL>(o, best_inl, V, nin, dadd(d, h), ray, cref, lane, gmask, scalar_mode);
    const double gm = tri_grad<G, OPL>(o, best_inl, V, nin, dsub(d, h), ray, cref, lane, gmask, scalar_mode);
    const double hess = ddiv(dsub(gp, gm), dmul(2.0, h));
    double step;
    if (hess > 0.0 && isfinite(hess) && (scalar_mode || isfinite(g))) {
      step = ddiv(-g, hess);
    } else {
      // vec: -sign(g) * 0.05 * |d| (sign(NaN) = NaN); scalar: -copysign(0.05 |d|, g)
      const double sg = isnan(g) ? g : (g > 0.0 ? 1.0 : (g < 0.0 ? -1.0 : 0.0));
      step = scalar_mode ? -copysign(dmul(0.05, fabs(d)), g) : dmul(dmul(-sg, 0.05), fabs(d));
    }
    bool accepted = false;
    double cand_cost = cost;
    for (int k = 0; k < 30; ++k) {
      const double cand = dadd(d, step);
      if (cand > 0.0) {
        const double cc = tri_cost<G, OPL>(o, best_inl, V, nin, cand, ray, cref, lane, gmask, scalar_mode);
        if (cc <= cost) {
          cand_cost = cc;
          accepted = true;
          break;
        }
      }
      step = dmul(step, 0.5);
    }
    if (!accepted) break;
    const bool converged = fabs(step) < dmul(cfg.refine_tol, fmax(fabs(d), 1e-300));
    d = dadd(d, step);
    cost = cand_cost;
    if (converged) break;
  }
  d_out = d;
  return best;
}

template <typename T>
__device__ __forceinline__ double ld(const void* p, int64_t i) {
  return (double)__ldg((const T*)p + i);
}

template <int G, int OPL>
__global__ void __launch_bounds__(kTriThreads, (OPL == 1 ? VL_TRI_MINB : 1)) k_tri_map(const TriMap* __restrict__ maps,
                                                         const TriView* __restrict__ views, int field_f64,
                                                         TriConfig cfg) {
  const TriMap& M = maps[blockIdx.y];
  const int lane = threadIdx.x % G;
  const int gbase = threadIdx.x & 31 & ~(G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  const int gpc = kTriThreads / G;  // pixels per CTA pass
  const int npix = M.grid_w * M.grid_h;
  const int V = M.nview;
  // groups are independent (group-masked shuffles/ballots only): no CTA-wide sync
  for (int p = blockIdx.x * gpc + threadIdx.x / G; p < npix; p += gridDim.x * gpc) {
    const int row = p / M.grid_w, col = p - row * M.grid_w;
    // reference ray through the cell centre (depthbuild.py:312-320)
    const double u = dmul(dadd((double)col, 0.5), M.sx), v = dmul(dadd((double)row, 0.5), M.sy);
    double k[3] = {ddiv(dsub(u, M.cx), M.fx), ddiv(dsub(v, M.cy), M.fy), 1.0};
    const double kn = sqrt(sum3(dmul(k[0], k[0]), dmul(k[1], k[1]), 1.0));
#pragma unroll
    for (int i = 0; i < 3; ++i) k[i] = ddiv(k[i], kn);
    double ray[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {  // k @ R  (rays = k @ ref_R_t.T)
      const double col3[3] = {M.R[i], M.R[3 + i], M.R[6 + i]};
      ray[i] = matmul3(k, col3);
    }
    LaneObs<OPL> o;
#pragma unroll
    for (int s = 0; s < OPL; ++s) {
      const int vi = s * G + lane;
      o.ok[s] = o.hok[s] = false;
      o.conf[s] = o.D[s] = 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i) o.b[s][i] = o.c[s][i] = 0.0;
      if (vi < V) {
        const TriView& W = views[M.view0 + vi];
        double tx, ty, cf;
        if (field_f64) {
          tx = ld<double>(W.targets, 2 * (int64_t)p);
          ty = ld<double>(W.targets, 2 * (int64_t)p + 1);
          cf = ld<double>(W.confidence, p);
        } else {
          tx = ld<float>(W.targets, 2 * (int64_t)p);
          ty = ld<float>(W.targets, 2 * (int64_t)p + 1);
          cf = ld<float>(W.confidence, p);
        }
        const bool ok = cf >= cfg.conf_thr && cf > 0.0;
        o.ok[s] = ok;
        o.conf[s] = cf;
        for (int i = 0; i < 3; ++i) o.c[s][i] = W.center[i];
        if (ok) view_bearing(W.rt, W.fx, W.fy, W.cx, W.cy, tx, ty, o.b[s]);
        hypothesis(ray, M.center, o.b[s], o.c[s], ok, o.D[s], o.hok[s]);
      }
    }
    double d = 0.0;
    const int n = tri_solve<G, OPL>(o, V, ray, M.center, cfg, lane, gmask, gbase, false, d);
    if (lane == 0) {
      M.depth[p] = n ? (float)ddiv(d, kn) : 0.0f;
      M.valid[p] = n ? 1 : 0;
    }
  }
}

template <int G, int OPL>
__global__ void __launch_bounds__(kTriThreads) k_tri_rays(const TriProblem* __restrict__ probs, int nprob,
                                                          const TriObs* __restrict__ obs, TriConfig cfg,
                                                          double* depth_out, int* count_out, double* hyp_out) {
  const int lane = threadIdx.x % G;
  const int gbase = threadIdx.x & 31 & ~(G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  const int gpc = kTriThreads / G;
  for (int p = blockIdx.x * gpc + threadIdx.x / G; p < nprob; p += gridDim.x * gpc) {
    const TriProblem& P = probs[p];
    const int V = P.nobs;
    LaneObs<OPL> o;
#pragma unroll
    for (int s = 0; s < OPL; ++s) {
      const int vi = s * G + lane;
      o.ok[s] = o.hok[s] = false;
      o.conf[s] = o.D[s] = 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i) o.b[s][i] = o.c[s][i] = 0.0;
      if (vi < V) {
        const TriObs& W = obs[P.obs0 + vi];
        o.ok[s] = true;  // triangulate_pixel: observations are confidence-filtered already
        o.conf[s] = W.confidence;
        for (int i = 0; i < 3; ++i) o.c[s][i] = W.center[i];
        view_bearing(W.rt, W.fx, W.fy, W.cx, W.cy, W.target[0], W.target[1], o.b[s]);
        hypothesis(P.ray, P.center, o.b[s], o.c[s], true, o.D[s], o.hok[s]);
        if (hyp_out) hyp_out[P.obs0 + vi] = o.hok[s] ? o.D[s] : CUDART_NAN;
      }
    }
    double d = 0.0;
    const int n = V > 0 ? tri_solve<G, OPL>(o, V, P.ray, P.center, cfg, lane, gmask, gbase, true, d) : 0;
    if (lane == 0) {
      depth_out[p] = n ? d : CUDART_NAN;
      count_out[p] = n;
    }
  }
}

// One pixel per warp: the Newton refinement diverges across pixels, so
// packing several pixels in a warp serialises them (measured, V=20, 441k px:
// G=32 7.8 ms, G=16 17.7 ms, G=8 21.5 ms).
static void pick(int maxv, int& G, int& OPL) {
  G = 32;
  OPL = std::max(1, (maxv + 31) / 32);
  if (const char* e = getenv("VISLOC_TRI_G")) {  // tuning override: lanes per pixel (8, 16, 32)
    const int g = atoi(e);
    if (g == 8 || g == 16 || g == 32) {
      G = g;
      OPL = std::max(1, (maxv + g - 1) / g);
      if (OPL > 4) G = 32, OPL = (maxv + 31) / 32;
    }
  }
}

#define VL_TRI_CASE(KERNEL, GG, OO, GRID, ...) \
  else if (G == GG && OPL == OO) KERNEL<GG, OO><<<GRID, kTriThreads, 0, st>>>(__VA_ARGS__);
#define VL_TRI_DISPATCH(KERNEL, GRID, ...)                                                      \
  do {                                                                                          \
    if (false) {}                                                                               \
    VL_TRI_CASE(KERNEL, 8, 1, GRID, __VA_ARGS__) VL_TRI_CASE(KERNEL, 8, 2, GRID, __VA_ARGS__)    \
    VL_TRI_CASE(KERNEL, 8, 3, GRID, __VA_ARGS__) VL_TRI_CASE(KERNEL, 8, 4, GRID, __VA_ARGS__)    \
    VL_TRI_CASE(KERNEL, 16, 1, GRID, __VA_ARGS__) VL_TRI_CASE(KERNEL, 16, 2, GRID, __VA_ARGS__)  \
    VL_TRI_CASE(KERNEL, 16, 3, GRID, __VA_ARGS__) VL_TRI_CASE(KERNEL, 16, 4, GRID, __VA_ARGS__)  \
    VL_TRI_CASE(KERNEL, 32, 1, GRID, __VA_ARGS__) VL_TRI_CASE(KERNEL, 32, 2, GRID, __VA_ARGS__)  \
    VL_TRI_CASE(KERNEL, 32, 3, GRID, __VA_ARGS__) VL_TRI_CASE(KERNEL, 32, 4, GRID, __VA_ARGS__)  \
  } while (0)

int launch_tri_maps(const TriMap* d_maps, int nmap, int max_pix, int max_views, const TriView* d_views, int f64,
                    const TriConfig& cfg, int num_sms, cudaStream_t st) {
  int G, OPL;
  pick(max_views, G, OPL);
  const int gpc = kTriThreads / G;
  const int want = (max_pix + gpc - 1) / gpc;
  const int gx = std::max(1, std::min(want, (num_sms * 8 + nmap - 1) / nmap));
  int launches = 0;
  for (int m0 = 0; m0 < nmap; m0 += 65535) {
    dim3 grid(gx, std::min(65535, nmap - m0));
    VL_TRI_DISPATCH(k_tri_map, grid, d_maps + m0, d_views, f64, cfg);
    ++launches;
  }
  return launches;
}

int launch_tri_rays(const TriProblem* d_probs, int nprob, int max_obs, const TriObs* d_obs, const TriConfig& cfg,
                    double* depth_out, int* count_out, double* hyp_out, int num_sms, cudaStream_t st) {
  int G, OPL;
  pick(max_obs, G, OPL);
  const int gpc = kTriThreads / G;
  const int gx = std::max(1, std::min((nprob + gpc - 1) / gpc, num_sms * 8));
  VL_TRI_DISPATCH(k_tri_rays, gx, d_probs, nprob, d_obs, cfg, depth_out, count_out, hyp_out);
  return 1;
}

}  // namespace vl
