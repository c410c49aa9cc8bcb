"""P3P minimal solver restated from the reference (fp64, numpy).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``pkg/src/visloc/p3p.py``:

* degeneracy gate — :91-98 (coincident / collinear points, |cos| >= 1);
* law-of-cosines quadrics reduced to a resultant quartic in v = s3/s1 —
  :108-141;
* per-sample ``np.roots`` (LAPACK geev on the companion matrix), keep roots
  with |Im| <= 1e-6 (1 + |Re|) and Re > 0, ascending — :147-166;
* u from the linear relation, or both branches of the first quadratic when
  the relation degenerates — ``_distance_triples`` :206-231;
* 12 Newton steps on the three quadrics, SVD Procrustes with det fix,
  bearing-residual contract <= 1e-8 rad — ``_poses_from_distances_batch``
  :234-306;
* per-sample dedup (||dR|| < 1e-6, ||dt|| < 1e-6 sqrt(scale2)), <= 4 kept —
  :168-199.
"""

from __future__ import annotations

import numpy as np

BEARING_TOL = 1e-8
COLLINEAR_TOL = 1e-9
DEDUP_TOL = 1e-6
NEWTON_ITERS = 12


def _sample_terms(f, P):
    a2 = ((P[:, 1] - P[:, 2]) ** 2).sum(-1)
    b2 = ((P[:, 0] - P[:, 2]) ** 2).sum(-1)
    c2 = ((P[:, 0] - P[:, 1]) ** 2).sum(-1)
    ca = (f[:, 1] * f[:, 2]).sum(-1)
    cb = (f[:, 0] * f[:, 2]).sum(-1)
    cg = (f[:, 0] * f[:, 1]).sum(-1)
    return a2, b2, c2, ca, cb, cg


def _gate(P, a2, b2, c2, ca, cb, cg):
    e1 = P[:, 1] - P[:, 0]
    e2 = P[:, 2] - P[:, 0]
    area = np.linalg.norm(np.cross(e1, e2), axis=-1)
    big = np.maximum(np.maximum(a2, b2), c2)
    small = np.minimum(np.minimum(a2, b2), c2)
    return ((big > 0) & (small > 1e-24 * big)
            & (area > COLLINEAR_TOL * np.linalg.norm(e1, axis=-1) * np.linalg.norm(e2, axis=-1))
            & (np.abs(ca) < 1.0) & (np.abs(cb) < 1.0) & (np.abs(cg) < 1.0)), big


def quartic_coeffs(a2, b2, c2, ca, cb, cg):
    """Resultant of u^2 + p1 u + q1(v) and u^2 + p2(v) u + q2(v); highest power first."""
    with np.errstate(divide="ignore", invalid="ignore"):
        ib = 1.0 / np.where(b2 > 0, b2, 1.0)
    # q1(v) = -(c2 (1 + v^2 - 2 v cb) - b2)/b2 ; q2(v) = (b2 v^2 - a2 (1 + v^2 - 2 v cb))/b2
    q10, q11, q12 = -(c2 - b2) * ib, -(-2.0 * c2 * cb) * ib, -c2 * ib
    q20, q21, q22 = -a2 * ib, 2.0 * a2 * cb * ib, (b2 - a2) * ib
    d0, d1, d2 = q20 - q10, q21 - q11, q22 - q12
    e0, e1 = -2.0 * cg, 2.0 * ca          # (p1 - p2)(v) = e0 + e1 v
    g0, g1, g2 = e0 * e0, 2 * e0 * e1, e1 * e1
    k4 = d2 * d2 + q12 * g2
    k3 = 2 * d1 * d2 + e0 * (d2 * e1) + (q11 * g2 + q12 * g1)
    k2 = (d1 * d1 + 2 * d0 * d2) + e0 * (d1 * e1 + d2 * e0) + (q10 * g2 + q11 * g1 + q12 * g0)
    k1 = 2 * d0 * d1 + e0 * (d0 * e1 + d1 * e0) + (q10 * g1 + q11 * g0)
    k0 = d0 * d0 + e0 * (d0 * e0) + q10 * g0
    return np.stack([k4, k3, k2, k1, k0], axis=-1)


def real_positive_roots(coeffs) -> list[float]:
    mx = np.max(np.abs(coeffs))
    if not np.isfinite(mx) or mx == 0:
        return []
    r = np.roots(coeffs / mx)
    return sorted(float(z.real) for z in r if abs(z.imag) <= 1e-6 * (1.0 + abs(z.real)) and z.real > 0)


def distance_triples(vs, a2, b2, c2, ca, cb, cg):
    out = []
    for v in vs:
        den = 1.0 + v * v - 2.0 * v * cb
        if den <= 0:
            continue
        s1 = np.sqrt(b2 / den)
        q1v = -((c2 * den - b2) / b2)
        q2v = (b2 * v * v - a2 * den) / b2
        pd = -2.0 * cg + 2.0 * v * ca
        if abs(pd) > 1e-10:
            us = [(q2v - q1v) / pd]
        else:
            disc = cg * cg - q1v
            if disc < 0:
                continue
            r = np.sqrt(disc)
            us = [cg + r, cg - r]
        out.extend([s1, u * s1, v * s1] for u in us if u > 0)
    return out


def polish_and_align(s, f, P, a2, b2, c2, ca, cb, cg):
    """Newton on the quadrics, Procrustes, contract check (stacked candidates)."""
    C = s.shape[0]
    scale2 = np.maximum(np.maximum(a2, b2), c2)
    s = s.copy()
    ok = np.ones(C, dtype=bool)
    for _ in range(NEWTON_ITERS):
        x, y, z = s[:, 0], s[:, 1], s[:, 2]
        res = np.stack([x * x + y * y - 2 * x * y * cg - c2,
                        x * x + z * z - 2 * x * z * cb - b2,
                        y * y + z * z - 2 * y * z * ca - a2], -1)
        live = ok & (np.abs(res).max(-1) >= 1e-14 * scale2)
        if not live.any():
            break
        zero = np.zeros(C)
        J = np.stack([np.stack([2 * x - 2 * y * cg, 2 * y - 2 * x * cg, zero], -1),
                      np.stack([2 * x - 2 * z * cb, zero, 2 * z - 2 * x * cb], -1),
                      np.stack([zero, 2 * y - 2 * z * ca, 2 * z - 2 * y * ca], -1)], 1)
        dJ = np.linalg.det(J)
        can = live & (np.abs(dJ) > 1e-300) & np.isfinite(dJ)
        ok &= ~(live & ~can)
        if not can.any():
            break
        step = np.zeros_like(s)
        step[can] = np.linalg.solve(J[can], -res[can][..., None])[..., 0]
        s = s + step
        ok &= ~(can & (np.any(~np.isfinite(s), -1) | np.any(s <= 0, -1)))
        s[~ok] = 1.0
    Y = s[:, :, None] * f
    Pm, Ym = P.mean(1), Y.mean(1)
    Hm = np.einsum("cni,cnj->cij", P - Pm[:, None], Y - Ym[:, None])
    U, _, Vt = np.linalg.svd(Hm)
    V = Vt.transpose(0, 2, 1)
    sgn = np.sign(np.linalg.det(np.einsum("cij,ckj->cik", V, U)))
    D = np.zeros((C, 3, 3))
    D[:, 0, 0] = D[:, 1, 1] = 1.0
    D[:, 2, 2] = sgn
    R = np.einsum("cij,cjk,clk->cil", V, D, U)
    t = Ym - np.einsum("cij,cj->ci", R, Pm)
    pred = np.einsum("cij,cnj->cni", R, P) + t[:, None, :]
    nr = np.linalg.norm(pred, axis=-1)
    front = np.all(nr > 0, -1)
    pred = pred / np.where(nr > 0, nr, 1.0)[..., None]
    ang = np.arctan2(np.linalg.norm(np.cross(pred, f), axis=-1), (pred * f).sum(-1))
    return R, t, ok & front & (ang.max(-1) <= BEARING_TOL)


def p3p_batch(bearings, points):
    """(R (M,3,3), t (M,3), sample (M,)) ordered by sample then ascending root."""
    f = np.asarray(bearings, dtype=np.float64)
    P = np.asarray(points, dtype=np.float64)
    a2, b2, c2, ca, cb, cg = _sample_terms(f, P)
    good, scale2 = _gate(P, a2, b2, c2, ca, cb, cg)
    quart = quartic_coeffs(a2, b2, c2, ca, cb, cg)
    owner, trip = [], []
    for i in np.nonzero(good)[0]:
        vs = real_positive_roots(quart[i])
        for s in distance_triples(vs, a2[i], b2[i], c2[i], ca[i], cb[i], cg[i]):
            owner.append(i)
            trip.append(s)
    empty = (np.zeros((0, 3, 3)), np.zeros((0, 3)), np.zeros(0, dtype=np.int64))
    if not owner:
        return empty
    idx = np.asarray(owner, dtype=np.int64)
    R, t, ok = polish_and_align(np.asarray(trip, dtype=np.float64), f[idx], P[idx],
                                a2[idx], b2[idx], c2[idx], ca[idx], cb[idx], cg[idx])
    keepR, keept, keepi = [], [], []
    per: dict[int, list] = {}
    for c in np.nonzero(ok)[0]:
        i = int(idx[c])
        lst = per.setdefault(i, [])
        if len(lst) >= 4:
            continue
        tol_t = DEDUP_TOL * np.sqrt(scale2[i])
        if any(np.linalg.norm(R[c] - Rk) < DEDUP_TOL and np.linalg.norm(t[c] - tk) < tol_t
               for Rk, tk in lst):
            continue
        lst.append((R[c], t[c]))
        keepR.append(R[c])
        keept.append(t[c])
        keepi.append(i)
    if not keepR:
        return empty
    return np.stack(keepR), np.stack(keept), np.asarray(keepi, dtype=np.int64)
