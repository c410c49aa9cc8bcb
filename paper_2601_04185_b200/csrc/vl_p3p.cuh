// fp64 P3P minimal solver building blocks, register resident.
//
// Same contract as pkg/src/visloc/p3p.py (p3p_solve_batch :57-203):
//  * degeneracy gate (:91-98);
//  * resultant quartic in v = s3/s1 with the reference's coefficient
//    assembly (:108-141), so the polynomial is bit-identical;
//  * real positive roots with |Im| <= 1e-6 (1 + |Re|), ascending (:147-166) —
//    all four complex roots are found with Aberth-Ehrlich iterations seeded
//    from the Newton polygon (instead of a LAPACK companion-matrix eigensolve)
//    and stopped once |p(z)| is at the rounding-error level of the
//    evaluation, which is where geev's roots sit too;
//  * u from the linear relation or both quadratic branches (:206-231);
//  * 12 Newton steps on the three law-of-cosines quadrics (:245-277);
//  * orthogonal Procrustes (:279-293): with three points both centred point
//    sets are planar, so the SVD solution R = V D U^T equals "map the world
//    triangle's plane frame onto the camera triangle's plane frame, then the
//    closed-form 2-D Procrustes rotation in that plane" — evaluated here
//    without an iterative SVD;
//  * bearing-residual contract <= 1e-8 rad and positive depths (:295-305);
//  * per-sample dedup (||dR||_F < 1e-6, ||dt|| < 1e-6 sqrt(scale2)), <= 4.
#pragma once
#include "vl_common.cuh"

namespace vl {

constexpr double kBearingTol = 1e-8;
constexpr double kCollinearTol = 1e-9;
constexpr double kDedupTol = 1e-6;
constexpr int kNewtonIters = 12;
constexpr int kMaxCand = 8;  // 4 roots x 2 branches
constexpr double kEps = 2.220446049250313e-16;

// Per-sample geometry shared by root finding and candidate polishing.
struct P3PGeo {
  double f[9], P[9];
  double a2, b2, c2, ca, cb, cg, scale2;
};

VL_HD void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
VL_HD double dot3(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
VL_HD double nrm3(const double* a) { return sqrt(dot3(a, a)); }

// Gate + quartic coefficients (highest power first).  Returns false for a
// degenerate sample.
VL_HD bool p3p_setup(const double* f, const double* P, P3PGeo& g, double* quart) {
  for (int i = 0; i < 9; ++i) {
    g.f[i] = f[i];
    g.P[i] = P[i];
  }
  double d12[3], d02[3], d01[3], e1v[3], e2v[3], cr[3];
  for (int i = 0; i < 3; ++i) {
    d12[i] = P[3 + i] - P[6 + i];
    d02[i] = P[i] - P[6 + i];
    d01[i] = P[i] - P[3 + i];
    e1v[i] = P[3 + i] - P[i];
    e2v[i] = P[6 + i] - P[i];
  }
  const double a2 = dot3(d12, d12), b2 = dot3(d02, d02), c2 = dot3(d01, d01);
  const double ca = dot3(f + 3, f + 6), cb = dot3(f, f + 6), cg = dot3(f, f + 3);
  cross3(e1v, e2v, cr);
  const double scale2 = fmax(fmax(a2, b2), c2);
  const double smin = fmin(fmin(a2, b2), c2);
  g.a2 = a2;
  g.b2 = b2;
  g.c2 = c2;
  g.ca = ca;
  g.cb = cb;
  g.cg = cg;
  g.scale2 = scale2;
  const bool ok = (scale2 > 0) && (smin > 1e-24 * scale2) &&
                  (nrm3(cr) > kCollinearTol * nrm3(e1v) * nrm3(e2v)) && (fabs(ca) < 1.0) &&
                  (fabs(cb) < 1.0) && (fabs(cg) < 1.0);
  if (!ok) return false;
  // quartic coefficients, assembled exactly like p3p.py:108-141
  const double rb = 1.0 / (b2 > 0 ? b2 : 1.0);
  const double q10 = -(c2 - b2) * rb, q11 = -(-2.0 * c2 * cb) * rb, q12 = -c2 * rb;
  const double q20 = -a2 * rb, q21 = 2.0 * a2 * cb * rb, q22 = (b2 - a2) * rb;
  const double d0 = q20 - q10, d1 = q21 - q11, d2 = q22 - q12;
  const double e0 = -2.0 * cg, e1 = 2.0 * ca;
  const double g0 = e0 * e0, g1 = 2 * e0 * e1, g2 = e1 * e1;
  quart[0] = d2 * d2 + q12 * g2;
  quart[1] = 2 * d1 * d2 + e0 * (d2 * e1) + (q11 * g2 + q12 * g1);
  quart[2] = (d1 * d1 + 2 * d0 * d2) + e0 * (d1 * e1 + d2 * e0) + (q10 * g2 + q11 * g1 + q12 * g0);
  quart[3] = 2 * d0 * d1 + e0 * (d0 * e1 + d1 * e0) + (q10 * g1 + q11 * g0);
  quart[4] = d0 * d0 + e0 * (d0 * e0) + q10 * g0;
  return true;
}

// Ferrari / resolvent-cubic approximations of the four roots of the monic
// quartic x^4 + b3 x^3 + b2 x^2 + b1 x + b0 (b[k] = coefficient of x^k).
// Only a starting point: the Aberth iterations below polish (and repair) it.
VL_HD bool ferrari_init(const double* b, double* zr, double* zi) {
  const double A = b[3], B = b[2], Cc = b[1], D = b[0];
  const double A2 = A * A;
  const double p = B - 0.375 * A2;
  const double q = Cc - 0.5 * A * B + 0.125 * A2 * A;
  const double r = D - 0.25 * A * Cc + 0.0625 * A2 * B - 0.01171875 * A2 * A2;
  // resolvent m^3 + p m^2 + (p^2/4 - r) m - q^2/8 = 0: largest real root
  const double a = p, bb = 0.25 * p * p - r, cc = -0.125 * q * q;
  const double Q = (a * a - 3.0 * bb) / 9.0, R = (2.0 * a * a * a - 9.0 * a * bb + 27.0 * cc) / 54.0;
  double m;
  if (R * R < Q * Q * Q) {
    const double sq = sqrt(Q);
    const double th = acos(fmin(fmax(R / (sq * sq * sq), -1.0), 1.0));
    m = -2.0 * sq * cos(th / 3.0) - a / 3.0;  // k = 0 gives the largest root
    m = fmax(m, -2.0 * sq * cos((th + 6.283185307179586) / 3.0) - a / 3.0);
    m = fmax(m, -2.0 * sq * cos((th - 6.283185307179586) / 3.0) - a / 3.0);
  } else {
    const double Aa = -copysign(cbrt(fabs(R) + sqrt(R * R - Q * Q * Q)), R);
    const double Bb = (Aa != 0.0) ? Q / Aa : 0.0;
    m = (Aa + Bb) - a / 3.0;
  }
  for (int it = 0; it < 2; ++it) {  // Newton polish of m
    const double f = ((m + a) * m + bb) * m + cc, fp = (3.0 * m + 2.0 * a) * m + bb;
    if (fp != 0.0) m -= f / fp;
  }
  const double sh = 0.25 * A;
  if (!(m > 1e-14 * (fabs(p) + 1e-300))) {
    // (near-)biquadratic: y^2 = (-p +- sqrt(p^2 - 4r)) / 2
    const double dsc = p * p - 4.0 * r;
    double wr[2], wi[2];
    if (dsc >= 0) {
      const double s = sqrt(dsc);
      wr[0] = 0.5 * (-p + s);
      wr[1] = 0.5 * (-p - s);
      wi[0] = wi[1] = 0.0;
    } else {
      wr[0] = wr[1] = -0.5 * p;
      wi[0] = 0.5 * sqrt(-dsc);
      wi[1] = -wi[0];
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // complex square roots of w
      const double mod = sqrt(wr[k] * wr[k] + wi[k] * wi[k]);
      double sr = sqrt(fmax(0.5 * (mod + wr[k]), 0.0));
      double si = sqrt(fmax(0.5 * (mod - wr[k]), 0.0));
      if (wi[k] < 0) si = -si;
      zr[2 * k] = sr - sh;
      zi[2 * k] = si;
      zr[2 * k + 1] = -sr - sh;
      zi[2 * k + 1] = -si;
    }
  } else {
    const double s = sqrt(2.0 * m);
    const double h = 0.5 * p + m, g = q / (2.0 * s);
    // y^2 - s y + (h + g) = 0 and y^2 + s y + (h - g) = 0
    const double c0[2] = {h + g, h - g};
    const double sg[2] = {s, -s};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double dsc = sg[k] * sg[k] - 4.0 * c0[k];
      if (dsc >= 0) {
        const double sd = sqrt(dsc);
        zr[2 * k] = 0.5 * (sg[k] + sd) - sh;
        zr[2 * k + 1] = 0.5 * (sg[k] - sd) - sh;
        zi[2 * k] = zi[2 * k + 1] = 0.0;
      } else {
        const double sd = sqrt(-dsc);
        zr[2 * k] = zr[2 * k + 1] = 0.5 * sg[k] - sh;
        zi[2 * k] = 0.5 * sd;
        zi[2 * k + 1] = -0.5 * sd;
      }
    }
  }
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 4; ++k) ok &= isfinite(zr[k]) && isfinite(zi[k]);
  // Aberth needs distinct starting points
  if (ok) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int j = k + 1; j < 4; ++j)
        if (zr[k] == zr[j] && zi[k] == zi[j]) {
          const double bump = 1e-7 * (1.0 + fabs(zr[k]));
          zi[j] += (j - k) * bump;
        }
  }
  return ok;
}

// Real positive roots (ascending) of sum_k c[k] v^(4-k); returns the count.
// Mirrors np.roots' degree handling: exact leading/trailing zeros stripped,
// zero roots never count (Re > 0 required).
VL_HD_BIG int quartic_real_pos_roots(const double* c_in, double* out) {
  double mx = 0;
#pragma unroll
  for (int k = 0; k < 5; ++k) mx = fmax(mx, fabs(c_in[k]));
  if (!isfinite(mx) || mx == 0) return 0;
  double c[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) c[k] = c_in[k] / mx;
  // every array below is indexed with compile-time indices only, so it stays
  // in registers (a runtime index moves the array to local memory)
  int lead = 4;  // first nonzero of c[0..3], else 4
#pragma unroll
  for (int k = 3; k >= 0; --k)
    if (c[k] != 0) lead = k;
  int last = lead;  // last nonzero above lead
#pragma unroll
  for (int k = 0; k < 5; ++k)
    if (k > lead && c[k] != 0) last = k;
  const int d = last - lead;
  if (d <= 0) return 0;
  // ascending monic coefficients b[k] of z^k (k <= d), zero-padded to 5
  // b[k] = c[last - k] / c[lead]: one static-index branch per `last` (a
  // select over j == last - k is turned back into an indexed local load)
  const double clead = lead == 0 ? c[0] : lead == 1 ? c[1] : lead == 2 ? c[2] : c[3];
  const double il = 1.0 / clead;
  double b[5];
#define VL_P3P_SHIFT(L)                                                     \
  _Pragma("unroll") for (int k = 0; k < 5; ++k) b[k] = (k <= d && k <= L) ? c[(L - k) < 0 ? 0 : (L - k)] * il : 0.0;
  switch (last) {
    case 4: VL_P3P_SHIFT(4) break;
    case 3: VL_P3P_SHIFT(3) break;
    case 2: VL_P3P_SHIFT(2) break;
    default: VL_P3P_SHIFT(1) break;
  }
#undef VL_P3P_SHIFT
  double zr[4], zi[4];
  bool conv[4];
  if (d == 1) {
    zr[0] = -b[0];
    zi[0] = 0.0;
  } else {
    const bool seeded = (d == 4) && ferrari_init(b, zr, zi);
    if (!seeded) {
    // Newton-polygon initial radii: upper convex hull of (k, log|b_k|).
    int hk[5];
    float hl[5];
    int nh = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (k > d || b[k] == 0) continue;
      const float lk = logf((float)fabs(b[k]));
      while (nh >= 2) {
        const float cr = (float)(hk[nh - 1] - hk[nh - 2]) * (lk - hl[nh - 2]) -
                         (hl[nh - 1] - hl[nh - 2]) * (float)(k - hk[nh - 2]);
        if (cr >= 0.f) --nh;
        else break;
      }
      hk[nh] = k;
      hl[nh] = lk;
      ++nh;
    }
    int zc = 0;
    for (int s = 0; s + 1 < nh; ++s) {
      const int m = hk[s + 1] - hk[s];
      const float r = expf((hl[s] - hl[s + 1]) / (float)m);
      for (int j = 0; j < m && zc < d; ++j) {
        const float ang = 6.2831853f * (float)j / (float)m + 1.5707963f / (float)d + 0.4f * s + 0.3f;
        float sn, cs;
        sincosf(ang, &sn, &cs);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (t == zc) {
            zr[t] = (double)(r * cs);
            zi[t] = (double)(r * sn);
          }
        ++zc;
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (t >= zc && t < d) {  // defensive: the hull always covers degree d
        zr[t] = cos(1.0 + t);
        zi[t] = sin(1.0 + t);
      }
    }  // !seeded
#pragma unroll
    for (int k = 0; k < 4; ++k) conv[k] = (k >= d);
    for (int it = 0; it < 60; ++it) {
      bool all = true;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (conv[k]) continue;
        const double xr = zr[k], xi = zi[k];
        // Horner for p, p' and the rounding bound sum |b_j| |z|^j
        const double az = sqrt(xr * xr + xi * xi);
        double pr = b[4], pi = 0.0, dr = 0.0, di = 0.0, bnd = fabs(b[4]);
#pragma unroll
        for (int j = 3; j >= 0; --j) {
          if (j >= d) {
            pr = b[j];  // leading coefficient (monic 1 at j == d)
            bnd = fabs(b[j]);
            continue;
          }
          const double ndr = dr * xr - di * xi + pr, ndi = dr * xi + di * xr + pi;
          const double npr = pr * xr - pi * xi + b[j], npi = pr * xi + pi * xr;
          dr = ndr;
          di = ndi;
          pr = npr;
          pi = npi;
          bnd = bnd * az + fabs(b[j]);
        }
        if (sqrt(pr * pr + pi * pi) <= 8.0 * kEps * bnd) {
          conv[k] = true;
          continue;
        }
        // ratio = p / p'
        const double idd = 1.0 / (dr * dr + di * di);
        const double rr = (pr * dr + pi * di) * idd, ri = (pi * dr - pr * di) * idd;
        // S = sum_{j != k} 1 / (z_k - z_j)
        double sr = 0.0, si = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j == k || j >= d) continue;
          const double ur = xr - zr[j], ui = xi - zi[j];
          const double iu = 1.0 / (ur * ur + ui * ui);
          sr += ur * iu;
          si -= ui * iu;
        }
        // corr = ratio / (1 - ratio * S)
        const double er = 1.0 - (rr * sr - ri * si), ei = -(rr * si + ri * sr);
        const double ie = 1.0 / (er * er + ei * ei);
        const double cr_ = (rr * er + ri * ei) * ie, ci_ = (ri * er - rr * ei) * ie;
        if (!(isfinite(cr_) && isfinite(ci_))) {
          conv[k] = true;
          continue;
        }
        zr[k] = xr - cr_;
        zi[k] = xi - ci_;
        if (sqrt(cr_ * cr_ + ci_ * ci_) <= 4.0 * kEps * sqrt(zr[k] * zr[k] + zi[k] * zi[k])) conv[k] = true;
        else all = false;
      }
      if (all) break;
    }
  }
  // ascending real positive roots: 4-element sorting network, rejected
  // roots parked at +inf (equal values are interchangeable)
  int nr = 0;
  double w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool keep = k < d && fabs(zi[k]) <= 1e-6 * (1.0 + fabs(zr[k])) && zr[k] > 0;
    w[k] = keep ? zr[k] : HUGE_VAL;
    nr += keep ? 1 : 0;
  }
  auto cswap = [](double& a, double& b) {
    const double lo = fmin(a, b), hi = fmax(a, b);
    a = lo;
    b = hi;
  };
  cswap(w[0], w[1]);
  cswap(w[2], w[3]);
  cswap(w[0], w[2]);
  cswap(w[1], w[3]);
  cswap(w[1], w[2]);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k < nr) out[k] = w[k];
  return nr;
}

// Distance-triple candidates (s1, s2, s3) from the roots (p3p.py:206-231),
// in reference order.  Returns the count (<= 8); component j of candidate k
// is written to cand[k*stride + j*estride] unless cand is null (count only).
VL_HD_BIG int p3p_candidates(const P3PGeo& g, const double* vs, int nv, double* cand, int stride,
                             int estride = 1) {
  int nc = 0;
  auto put = [&](double a, double b, double c) {
    if (cand) {
      cand[stride * nc] = a;
      cand[stride * nc + estride] = b;
      cand[stride * nc + 2 * estride] = c;
    }
    ++nc;
  };
#pragma unroll
  for (int iv = 0; iv < 4; ++iv) {
    if (iv >= nv) break;
    const double v = vs[iv];
    const double den = 1.0 + v * v - 2.0 * v * g.cb;
    if (den <= 0) continue;
    const double s1 = sqrt(g.b2 / den);
    const double q1v = -((g.c2 * den - g.b2) / g.b2);
    const double q2v = (g.b2 * v * v - g.a2 * den) / g.b2;
    const double pd = -2.0 * g.cg + 2.0 * v * g.ca;
    if (fabs(pd) > 1e-10) {
      const double u = (q2v - q1v) / pd;
      if (u > 0) put(s1, u * s1, v * s1);
    } else {
      const double disc = g.cg * g.cg - q1v;
      if (disc < 0) continue;
      const double r = sqrt(disc);
      const double u0 = g.cg + r, u1 = g.cg - r;
      if (u0 > 0) put(s1, u0 * s1, v * s1);
      if (u1 > 0) put(s1, u1 * s1, v * s1);
    }
  }
  return nc;
}

// 3x3 solve with partial pivoting; returns false on an exactly zero pivot.
VL_HD bool solve3(const double* Ain, const double* bin, double* x) {
  double A[9], b[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) A[i] = Ain[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) b[i] = bin[i];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    int p = k;
#pragma unroll
    for (int i = k + 1; i < 3; ++i)
      if (fabs(A[3 * i + k]) > fabs(A[3 * p + k])) p = i;
    // branch-free row swap (keeps A in registers)
#pragma unroll
    for (int i = k + 1; i < 3; ++i) {
      if (p == i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double tmp = A[3 * k + j];
          A[3 * k + j] = A[3 * i + j];
          A[3 * i + j] = tmp;
        }
        const double tb = b[k];
        b[k] = b[i];
        b[i] = tb;
      }
    }
    if (A[3 * k + k] == 0) return false;
    const double inv = 1.0 / A[3 * k + k];
#pragma unroll
    for (int i = k + 1; i < 3; ++i) {
      const double fct = A[3 * i + k] * inv;
#pragma unroll
      for (int j = k; j < 3; ++j) A[3 * i + j] -= fct * A[3 * k + j];
      b[i] -= fct * b[k];
    }
  }
#pragma unroll
  for (int i = 2; i >= 0; --i) {
    double s = b[i];
#pragma unroll
    for (int j = i + 1; j < 3; ++j) s -= A[3 * i + j] * x[j];
    x[i] = s / A[3 * i + i];
  }
  return true;
}

VL_HD double det3(const double* J) {
  return J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
         J[2] * (J[3] * J[7] - J[4] * J[6]);
}

// Orthonormal frame (a, b, n) of the plane through three points.
VL_HD void plane_frame(const double* X0, const double* X1, const double* X2, double* a, double* b, double* n) {
  double e1[3], e2[3];
  for (int i = 0; i < 3; ++i) {
    e1[i] = X1[i] - X0[i];
    e2[i] = X2[i] - X0[i];
  }
  cross3(e1, e2, n);
  const double in = 1.0 / nrm3(n);
  const double ia = 1.0 / nrm3(e1);
  for (int i = 0; i < 3; ++i) {
    n[i] *= in;
    a[i] = e1[i] * ia;
  }
  cross3(n, a, b);
}

// Newton polish of one distance triple, then Procrustes and the bearing
// contract.  Returns false for an invalid candidate.
VL_HD_BIG bool p3p_polish(const P3PGeo& g, const double* s_in, double* R, double* t) {
  double s0 = s_in[0], s1 = s_in[1], s2 = s_in[2];
  for (int it = 0; it < kNewtonIters; ++it) {
    const double r0 = s0 * s0 + s1 * s1 - 2 * s0 * s1 * g.cg - g.c2;
    const double r1 = s0 * s0 + s2 * s2 - 2 * s0 * s2 * g.cb - g.b2;
    const double r2 = s1 * s1 + s2 * s2 - 2 * s1 * s2 * g.ca - g.a2;
    const double mr = fmax(fmax(fabs(r0), fabs(r1)), fabs(r2));
    if (!(mr >= 1e-14 * g.scale2)) break;  // converged (inactive)
    const double J[9] = {2 * s0 - 2 * s1 * g.cg, 2 * s1 - 2 * s0 * g.cg, 0.0,
                         2 * s0 - 2 * s2 * g.cb, 0.0,                    2 * s2 - 2 * s0 * g.cb,
                         0.0,                    2 * s1 - 2 * s2 * g.ca, 2 * s2 - 2 * s1 * g.ca};
    const double dj = det3(J);
    if (!(fabs(dj) > 1e-300 && isfinite(dj))) return false;
    const double rhs[3] = {-r0, -r1, -r2};
    double st[3];
    if (!solve3(J, rhs, st)) return false;
    s0 += st[0];
    s1 += st[1];
    s2 += st[2];
    if (!(isfinite(s0) && isfinite(s1) && isfinite(s2)) || s0 <= 0 || s1 <= 0 || s2 <= 0) return false;
  }
  const double* f = g.f;
  const double* P = g.P;
  double Y[9];
  for (int i = 0; i < 3; ++i) {
    Y[i] = s0 * f[i];
    Y[3 + i] = s1 * f[3 + i];
    Y[6 + i] = s2 * f[6 + i];
  }
  double Pm[3], Ym[3];
  for (int i = 0; i < 3; ++i) {
    // centroids: * (1/3) instead of / 3 (<= 1 ulp from numpy's mean; P3P parity is 1e-9)
    Pm[i] = ((P[i] + P[3 + i]) + P[6 + i]) * (1.0 / 3.0);
    Ym[i] = ((Y[i] + Y[3 + i]) + Y[6 + i]) * (1.0 / 3.0);
  }
  // Plane frames of both triangles; R = F_Y * Rot2(theta) * F_P^T with the
  // closed-form 2-D Procrustes angle of the centred in-plane coordinates.
  double aP[3], bP[3], nP[3], aY[3], bY[3], nY[3];
  plane_frame(P, P + 3, P + 6, aP, bP, nP);
  plane_frame(Y, Y + 3, Y + 6, aY, bY, nY);
  double sc = 0.0, ss = 0.0;
  for (int k = 0; k < 3; ++k) {
    double pc[3], yc[3];
    for (int i = 0; i < 3; ++i) {
      pc[i] = P[3 * k + i] - Pm[i];
      yc[i] = Y[3 * k + i] - Ym[i];
    }
    const double px = dot3(pc, aP), py = dot3(pc, bP);
    const double yx = dot3(yc, aY), yy = dot3(yc, bY);
    sc += px * yx + py * yy;
    ss += px * yy - py * yx;
  }
  const double ih = 1.0 / sqrt(sc * sc + ss * ss);
  const double cth = sc * ih, sth = ss * ih;
  // columns of the rotated camera frame: a' = c aY + s bY, b' = -s aY + c bY
  double ar[3], br[3];
  for (int i = 0; i < 3; ++i) {
    ar[i] = cth * aY[i] + sth * bY[i];
    br[i] = -sth * aY[i] + cth * bY[i];
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = ar[i] * aP[j] + br[i] * bP[j] + nY[i] * nP[j];
  for (int i = 0; i < 3; ++i) t[i] = Ym[i] - (R[3 * i] * Pm[0] + R[3 * i + 1] * Pm[1] + R[3 * i + 2] * Pm[2]);
  // contract: every bearing reproduced to 1e-8 rad, positive norms
  for (int k = 0; k < 3; ++k) {
    double pr[3];
    for (int i = 0; i < 3; ++i)
      pr[i] = (R[3 * i] * P[3 * k] + R[3 * i + 1] * P[3 * k + 1] + R[3 * i + 2] * P[3 * k + 2]) + t[i];
    // positive norm (sqrt(n2) > 0 <=> n2 > 0, NaN fails both)
    if (!(dot3(pr, pr) > 0)) return false;
    // ang = atan2(|pr x f|, pr . f) <= tol on the normalised pr.  Away from the
    // threshold the decision is taken on the unnormalised pr: the ratio |c| / d
    // does not depend on |pr| and the 1 % band dwarfs the rounding, so the
    // decision is identical; within the band the reference's normalised atan2
    // decides (atan is monotone and atan(x) <= x)
    {
      double cx[3];
      cross3(pr, f + 3 * k, cx);
      const double c = nrm3(cx), d = dot3(pr, f + 3 * k);
      if (d > 0.0 && c <= 0.99 * kBearingTol * d) continue;
      if (!(d > 0.0) || c >= 1.01 * kBearingTol * d) return false;
    }
    const double inr = 1.0 / nrm3(pr);
    for (int i = 0; i < 3; ++i) pr[i] *= inr;
    double cx[3];
    cross3(pr, f + 3 * k, cx);
    const double c = nrm3(cx), d = dot3(pr, f + 3 * k);
    if (!(d > 0.0)) return false;
    const double ang = atan2(c, d);
    if (!(ang <= kBearingTol)) return false;
  }
  return true;
}

VL_HD bool p3p_is_dup(const double* R, const double* t, const double* Rk, const double* tk, double ttol) {
  double dr = 0, dt = 0;
  for (int i = 0; i < 9; ++i) {
    const double e = R[i] - Rk[i];
    dr += e * e;
  }
  for (int i = 0; i < 3; ++i) {
    const double e = t[i] - tk[i];
    dt += e * e;
  }
  return sqrt(dr) < kDedupTol && sqrt(dt) < ttol;
}

// Whole-sample solve (sequential over candidates).  Returns the number of
// solutions written to Rs[k*9], ts[k*3] in reference order.
VL_HD int p3p_solve_one(const double* f, const double* P, double* Rs, double* ts) {
  P3PGeo g;
  double quart[5];
  if (!p3p_setup(f, P, g, quart)) return 0;
  double vs[4];
  const int nv = quartic_real_pos_roots(quart, vs);
  if (nv == 0) return 0;
  double cand[3 * kMaxCand];
  const int nc = p3p_candidates(g, vs, nv, cand, 3);
  const double ttol = kDedupTol * sqrt(g.scale2);
  int nsol = 0;
  for (int c = 0; c < nc && nsol < kMaxSolPerSample; ++c) {
    double R[9], t[3];
    if (!p3p_polish(g, cand + 3 * c, R, t)) continue;
    bool dup = false;
    for (int k = 0; k < nsol && !dup; ++k) dup = p3p_is_dup(R, t, Rs + 9 * k, ts + 3 * k, ttol);
    if (dup) continue;
    for (int i = 0; i < 9; ++i) Rs[9 * nsol + i] = R[i];
    for (int i = 0; i < 3; ++i) ts[3 * nsol + i] = t[i];
    ++nsol;
  }
  return nsol;
}

}  // namespace vl
