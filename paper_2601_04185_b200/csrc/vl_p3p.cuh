// Per-thread fp64 P3P minimal solver, register resident.
//
// Same contract as pkg/src/visloc/p3p.py (p3p_solve_batch :57-203):
//  * degeneracy gate (:91-98);
//  * resultant quartic in v = s3/s1 with the reference's coefficient
//    assembly (:108-141), so the polynomial is bit-identical;
//  * real positive roots with |Im| <= 1e-6 (1 + |Re|), ascending (:147-166) —
//    found here with Aberth-Ehrlich iterations seeded from the Newton
//    polygon instead of a LAPACK companion-matrix eigensolve;
//  * u from the linear relation or both quadratic branches (:206-231);
//  * 12 Newton steps on the three law-of-cosines quadrics (:245-277);
//  * orthogonal Procrustes R = V D U^T (:279-293) — computed with a one-sided
//    Jacobi SVD of the 3x3 cross-covariance; with three points the
//    covariance has rank 2 and V D U^T = v1u1' + v2u2' + (v1xv2)(u1xu2)';
//  * bearing-residual contract <= 1e-8 rad and positive depths (:295-305);
//  * per-sample dedup (||dR||_F < 1e-6, ||dt|| < 1e-6 sqrt(scale2)), <= 4.
#pragma once
#include "vl_common.cuh"

namespace vl {

constexpr double kBearingTol = 1e-8;
constexpr double kCollinearTol = 1e-9;
constexpr double kDedupTol = 1e-6;
constexpr int kNewtonIters = 12;

struct cplx {
  double re, im;
};
VL_HD cplx cmk(double r, double i) { return cplx{r, i}; }
VL_HD cplx cadd(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }
VL_HD cplx csub(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }
VL_HD cplx cmul(cplx a, cplx b) { return cplx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
VL_HD cplx cdiv(cplx a, cplx b) {
  // Smith's algorithm
  if (fabs(b.re) >= fabs(b.im)) {
    const double r = b.im / b.re, d = b.re + b.im * r;
    return cplx{(a.re + a.im * r) / d, (a.im - a.re * r) / d};
  }
  const double r = b.re / b.im, d = b.im + b.re * r;
  return cplx{(a.re * r + a.im) / d, (a.im * r - a.re) / d};
}
VL_HD double cabs_(cplx a) { return hypot(a.re, a.im); }

// Real positive roots (ascending) of sum_k c[k] v^(4-k); returns count.
// Mirrors np.roots' degree handling: exact leading/trailing zeros stripped,
// zero roots never count (Re > 0 required).
VL_HD int quartic_real_pos_roots(const double* c_in, double* out) {
  double mx = 0;
  for (int k = 0; k < 5; ++k) mx = fmax(mx, fabs(c_in[k]));
  if (!isfinite(mx) || mx == 0) return 0;  // non-finite or all-zero
  double c[5];
  for (int k = 0; k < 5; ++k) c[k] = c_in[k] / mx;
  int lead = 0;
  while (lead < 5 && c[lead] == 0) ++lead;
  int last = 4;
  while (last > lead && c[last] == 0) --last;
  const int d = last - lead;  // degree after stripping
  if (d <= 0) return 0;
  // ascending coefficients b[k] of z^k, monic
  double b[5];
  for (int k = 0; k <= d; ++k) b[k] = c[last - k] / c[lead];
  cplx z[4];
  if (d == 1) {
    z[0] = cmk(-b[0], 0.0);
  } else {
    // Newton-polygon initial radii (upper convex hull of (k, log|b_k|)).
    int hk[5];
    double hl[5];
    int nh = 0;
    for (int k = 0; k <= d; ++k) {
      if (b[k] == 0) continue;
      const double lk = log(fabs(b[k]));
      while (nh >= 2) {
        // pop if (hk[nh-2],hl[nh-2]) -> (hk[nh-1],hl[nh-1]) -> (k,lk) is not a right turn
        const double cr = (hk[nh - 1] - hk[nh - 2]) * (lk - hl[nh - 2]) -
                          (hl[nh - 1] - hl[nh - 2]) * (k - hk[nh - 2]);
        if (cr >= 0) --nh;
        else break;
      }
      hk[nh] = k;
      hl[nh] = lk;
      ++nh;
    }
    int zi = 0;
    for (int s = 0; s + 1 < nh; ++s) {
      const int m = hk[s + 1] - hk[s];
      const double r = exp((hl[s] - hl[s + 1]) / m);
      for (int j = 0; j < m && zi < d; ++j) {
        const double ang = 6.283185307179586 * j / m + 1.5707963267948966 / d + 0.4 * s + 0.3;
        z[zi++] = cmk(r * cos(ang), r * sin(ang));
      }
    }
    while (zi < d) {  // defensive: hull always covers degree d
      z[zi] = cmk(cos(1.0 + zi), sin(1.0 + zi));
      ++zi;
    }
    bool conv[4] = {false, false, false, false};
    for (int it = 0; it < 80; ++it) {
      bool all = true;
      for (int k = 0; k < d; ++k) {
        if (conv[k]) continue;
        // Horner for p and p'
        cplx p = cmk(b[d], 0.0), dp = cmk(0.0, 0.0);
        for (int j = d - 1; j >= 0; --j) {
          dp = cadd(cmul(dp, z[k]), p);
          p = cadd(cmul(p, z[k]), cmk(b[j], 0.0));
        }
        if (p.re == 0 && p.im == 0) {
          conv[k] = true;
          continue;
        }
        const cplx ratio = cdiv(p, dp);
        cplx s = cmk(0.0, 0.0);
        for (int j = 0; j < d; ++j)
          if (j != k) s = cadd(s, cdiv(cmk(1.0, 0.0), csub(z[k], z[j])));
        const cplx den = csub(cmk(1.0, 0.0), cmul(ratio, s));
        const cplx corr = cdiv(ratio, den);
        if (!(isfinite(corr.re) && isfinite(corr.im))) {
          conv[k] = true;
          continue;
        }
        z[k] = csub(z[k], corr);
        if (cabs_(corr) <= 4.0 * 2.220446049250313e-16 * cabs_(z[k])) conv[k] = true;
        else all = false;
      }
      if (all) break;
    }
  }
  int nr = 0;
  for (int k = 0; k < d; ++k) {
    if (fabs(z[k].im) <= 1e-6 * (1.0 + fabs(z[k].re)) && z[k].re > 0) {
      // insertion sort ascending
      int p = nr++;
      while (p > 0 && out[p - 1] > z[k].re) {
        out[p] = out[p - 1];
        --p;
      }
      out[p] = z[k].re;
    }
  }
  return nr;
}

// 3x3 solve with partial pivoting; returns false if singular.
VL_HD bool solve3(const double* Ain, const double* bin, double* x) {
  double A[9], b[3];
  for (int i = 0; i < 9; ++i) A[i] = Ain[i];
  for (int i = 0; i < 3; ++i) b[i] = bin[i];
  for (int k = 0; k < 3; ++k) {
    int p = k;
    for (int i = k + 1; i < 3; ++i)
      if (fabs(A[3 * i + k]) > fabs(A[3 * p + k])) p = i;
    if (A[3 * p + k] == 0) return false;
    if (p != k) {
      for (int j = 0; j < 3; ++j) {
        double tmp = A[3 * k + j];
        A[3 * k + j] = A[3 * p + j];
        A[3 * p + j] = tmp;
      }
      double tb = b[k];
      b[k] = b[p];
      b[p] = tb;
    }
    for (int i = k + 1; i < 3; ++i) {
      const double f = A[3 * i + k] / A[3 * k + k];
      for (int j = k; j < 3; ++j) A[3 * i + j] -= f * A[3 * k + j];
      b[i] -= f * b[k];
    }
  }
  for (int i = 2; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < 3; ++j) s -= A[3 * i + j] * x[j];
    x[i] = s / A[3 * i + i];
  }
  return true;
}

VL_HD double det3(const double* J) {
  return J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
         J[2] * (J[3] * J[7] - J[4] * J[6]);
}

VL_HD void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
VL_HD double dot3(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
VL_HD double nrm3(const double* a) { return sqrt(dot3(a, a)); }

// Orthogonal Procrustes: R maximising tr(R^T ...) for H = sum Pc Yc^T,
// R = V D U^T with H = U S V^T (one-sided Jacobi on H's columns).
VL_HD void procrustes_R(const double* H, double* R) {
  double A[9], V[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  for (int i = 0; i < 9; ++i) A[i] = H[i];
  for (int sweep = 0; sweep < 12; ++sweep) {
    double off = 0;
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      double al = 0, be = 0, ga = 0;
      for (int i = 0; i < 3; ++i) {
        al += A[3 * i + p] * A[3 * i + p];
        be += A[3 * i + q] * A[3 * i + q];
        ga += A[3 * i + p] * A[3 * i + q];
      }
      if (ga == 0) continue;
      const double sc = fabs(ga) / sqrt(al * be);
      if (!(sc > 1e-17)) continue;
      off = fmax(off, sc);
      const double zeta = (be - al) / (2.0 * ga);
      const double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
      const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
      for (int i = 0; i < 3; ++i) {
        const double ap = A[3 * i + p], aq = A[3 * i + q];
        A[3 * i + p] = cs * ap - sn * aq;
        A[3 * i + q] = sn * ap + cs * aq;
        const double vp = V[3 * i + p], vq = V[3 * i + q];
        V[3 * i + p] = cs * vp - sn * vq;
        V[3 * i + q] = sn * vp + cs * vq;
      }
    }
    if (off < 1e-15) break;
  }
  double sg[3];
  for (int k = 0; k < 3; ++k) sg[k] = sqrt(A[k] * A[k] + A[3 + k] * A[3 + k] + A[6 + k] * A[6 + k]);
  // indices of the two largest singular values
  int i1 = 0;
  for (int k = 1; k < 3; ++k)
    if (sg[k] > sg[i1]) i1 = k;
  int i2 = i1 == 0 ? 1 : 0;
  for (int k = 0; k < 3; ++k)
    if (k != i1 && sg[k] > sg[i2]) i2 = k;
  double u1[3], u2[3], v1[3], v2[3], u3[3], v3[3];
  for (int i = 0; i < 3; ++i) {
    u1[i] = A[3 * i + i1] / sg[i1];
    u2[i] = A[3 * i + i2] / sg[i2];
    v1[i] = V[3 * i + i1];
    v2[i] = V[3 * i + i2];
  }
  cross3(u1, u2, u3);
  cross3(v1, v2, v3);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = v1[i] * u1[j] + v2[i] * u2[j] + v3[i] * u3[j];
}

// Solve one minimal sample.  f, P: row-major (3 points x 3).  Returns the
// number of solutions written to Rs[k*9], ts[k*3] in reference order.
VL_HD int p3p_solve_one(const double* f, const double* P, double* Rs, double* ts) {
  double d12[3], d02[3], d01[3];
  for (int i = 0; i < 3; ++i) {
    d12[i] = P[3 + i] - P[6 + i];
    d02[i] = P[i] - P[6 + i];
    d01[i] = P[i] - P[3 + i];
  }
  const double a2 = dot3(d12, d12), b2 = dot3(d02, d02), c2 = dot3(d01, d01);
  const double ca = dot3(f + 3, f + 6), cb = dot3(f, f + 6), cg = dot3(f, f + 3);
  double e1v[3], e2v[3], cr[3];
  for (int i = 0; i < 3; ++i) {
    e1v[i] = P[3 + i] - P[i];
    e2v[i] = P[6 + i] - P[i];
  }
  cross3(e1v, e2v, cr);
  const double scale2 = fmax(fmax(a2, b2), c2);
  const double smin = fmin(fmin(a2, b2), c2);
  const bool ok = (scale2 > 0) && (smin > 1e-24 * scale2) &&
                  (nrm3(cr) > kCollinearTol * nrm3(e1v) * nrm3(e2v)) && (fabs(ca) < 1.0) &&
                  (fabs(cb) < 1.0) && (fabs(cg) < 1.0);
  if (!ok) return 0;

  // quartic coefficients, assembled exactly like p3p.py:108-141
  const double rb = 1.0 / (b2 > 0 ? b2 : 1.0);
  const double q10 = -(c2 - b2) * rb, q11 = -(-2.0 * c2 * cb) * rb, q12 = -c2 * rb;
  const double q20 = -a2 * rb, q21 = 2.0 * a2 * cb * rb, q22 = (b2 - a2) * rb;
  const double d0 = q20 - q10, d1 = q21 - q11, d2 = q22 - q12;
  const double e0 = -2.0 * cg, e1 = 2.0 * ca;
  const double g0 = e0 * e0, g1 = 2 * e0 * e1, g2 = e1 * e1;
  double quart[5];
  quart[0] = d2 * d2 + q12 * g2;
  quart[1] = 2 * d1 * d2 + e0 * (d2 * e1) + (q11 * g2 + q12 * g1);
  quart[2] = (d1 * d1 + 2 * d0 * d2) + e0 * (d1 * e1 + d2 * e0) + (q10 * g2 + q11 * g1 + q12 * g0);
  quart[3] = 2 * d0 * d1 + e0 * (d0 * e1 + d1 * e0) + (q10 * g1 + q11 * g0);
  quart[4] = d0 * d0 + e0 * (d0 * e0) + q10 * g0;

  double vs[4];
  const int nv = quartic_real_pos_roots(quart, vs);
  if (nv == 0) return 0;

  int nsol = 0;
  const double ttol = kDedupTol * sqrt(scale2);
  for (int iv = 0; iv < nv; ++iv) {
    const double v = vs[iv];
    const double den = 1.0 + v * v - 2.0 * v * cb;
    if (den <= 0) continue;
    const double s1 = sqrt(b2 / den);
    const double q1v = -((c2 * den - b2) / b2);
    const double q2v = (b2 * v * v - a2 * den) / b2;
    const double pd = -2.0 * cg + 2.0 * v * ca;
    double us[2];
    int nu = 0;
    if (fabs(pd) > 1e-10) {
      us[nu++] = (q2v - q1v) / pd;
    } else {
      const double disc = cg * cg - q1v;
      if (disc < 0) continue;
      const double r = sqrt(disc);
      us[nu++] = cg + r;
      us[nu++] = cg - r;
    }
    for (int iu = 0; iu < nu; ++iu) {
      const double u = us[iu];
      if (u <= 0) continue;
      if (nsol >= kMaxSolPerSample) return nsol;
      // ---- Newton polish of (s1, s2, s3)
      double s[3] = {s1, u * s1, v * s1};
      bool valid = true;
      for (int it = 0; it < kNewtonIters; ++it) {
        const double x = s[0], y = s[1], z = s[2];
        double r[3] = {x * x + y * y - 2 * x * y * cg - c2, x * x + z * z - 2 * x * z * cb - b2,
                       y * y + z * z - 2 * y * z * ca - a2};
        const double mr = fmax(fmax(fabs(r[0]), fabs(r[1])), fabs(r[2]));
        if (!(mr >= 1e-14 * scale2)) break;  // inactive (converged)
        const double J[9] = {2 * x - 2 * y * cg, 2 * y - 2 * x * cg, 0.0,
                             2 * x - 2 * z * cb, 0.0,                2 * z - 2 * x * cb,
                             0.0,                2 * y - 2 * z * ca, 2 * z - 2 * y * ca};
        const double dj = det3(J);
        if (!(fabs(dj) > 1e-300 && isfinite(dj))) {
          valid = false;
          break;
        }
        const double mrhs[3] = {-r[0], -r[1], -r[2]};
        double st[3];
        if (!solve3(J, mrhs, st)) {
          valid = false;
          break;
        }
        s[0] = x + st[0];
        s[1] = y + st[1];
        s[2] = z + st[2];
        if (!(isfinite(s[0]) && isfinite(s[1]) && isfinite(s[2])) || s[0] <= 0 || s[1] <= 0 ||
            s[2] <= 0) {
          valid = false;
          break;
        }
      }
      if (!valid) continue;
      // ---- Procrustes
      double Y[9];
      for (int n = 0; n < 3; ++n)
        for (int i = 0; i < 3; ++i) Y[3 * n + i] = s[n] * f[3 * n + i];
      double Pm[3], Ym[3];
      for (int i = 0; i < 3; ++i) {
        Pm[i] = ((P[i] + P[3 + i]) + P[6 + i]) / 3.0;
        Ym[i] = ((Y[i] + Y[3 + i]) + Y[6 + i]) / 3.0;
      }
      double H[9];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          double acc = 0;
          for (int n = 0; n < 3; ++n) acc += (P[3 * n + i] - Pm[i]) * (Y[3 * n + j] - Ym[j]);
          H[3 * i + j] = acc;
        }
      double R[9], t[3];
      procrustes_R(H, R);
      for (int i = 0; i < 3; ++i) t[i] = Ym[i] - (R[3 * i] * Pm[0] + R[3 * i + 1] * Pm[1] + R[3 * i + 2] * Pm[2]);
      // ---- contract: every bearing reproduced to 1e-8 rad, positive norms
      bool good = true;
      for (int n = 0; n < 3 && good; ++n) {
        double pr[3];
        for (int i = 0; i < 3; ++i)
          pr[i] = (R[3 * i] * P[3 * n] + R[3 * i + 1] * P[3 * n + 1] + R[3 * i + 2] * P[3 * n + 2]) + t[i];
        const double nr = nrm3(pr);
        if (!(nr > 0)) {
          good = false;
          break;
        }
        for (int i = 0; i < 3; ++i) pr[i] /= nr;
        double cx[3];
        cross3(pr, f + 3 * n, cx);
        const double ang = atan2(nrm3(cx), dot3(pr, f + 3 * n));
        if (!(ang <= kBearingTol)) good = false;
      }
      if (!good) continue;
      // ---- dedup against kept solutions of this sample
      bool dup = false;
      for (int k = 0; k < nsol && !dup; ++k) {
        double dr = 0, dt = 0;
        for (int i = 0; i < 9; ++i) {
          const double e = R[i] - Rs[9 * k + i];
          dr += e * e;
        }
        for (int i = 0; i < 3; ++i) {
          const double e = t[i] - ts[3 * k + i];
          dt += e * e;
        }
        if (sqrt(dr) < kDedupTol && sqrt(dt) < ttol) dup = true;
      }
      if (dup) continue;
      for (int i = 0; i < 9; ++i) Rs[9 * nsol + i] = R[i];
      for (int i = 0; i < 3; ++i) ts[3 * nsol + i] = t[i];
      ++nsol;
    }
  }
  return nsol;
}

}  // namespace vl
