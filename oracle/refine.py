"""LM / IRLS pose refinement restated from the reference (fp64, numpy).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``pkg/src/visloc/refine.py``: losses :43-77 (truncated rho = min(e2,
tau^2), weight 1[e2 < tau^2], behind tau^2; Cauchy rho = c^2/2 log1p(e2/c^2),
weight 0.5/(1+e2/c^2), behind inf), residuals :90-100, analytic Jacobian
:103-132, robust cost :135-149, LM schedule :164-230 (lambda 1e-6, 25
damping trials x10, accept on <=, lambda/3 floor 1e-12, gradient tol 1e-10,
relative cost tol 1e-12).
"""

from __future__ import annotations

import math

import numpy as np

from .geometry import apply_delta, q2R

TRUNCATED = "truncated"
CAUCHY = "cauchy"


def _rho(kind, scale, e2):
    s2 = scale * scale
    if kind == TRUNCATED:
        return np.minimum(e2, s2)
    return 0.5 * s2 * np.log1p(e2 / s2)


def _wt(kind, scale, e2):
    s2 = scale * scale
    if kind == TRUNCATED:
        return (e2 < s2).astype(np.float64)
    return 0.5 / (1.0 + e2 / s2)


def _behind(kind, scale):
    return scale * scale if kind == TRUNCATED else math.inf


def residuals(pose, X, px, intr):
    q, t = pose
    xc = X @ q2R(q).T + t
    z = xc[:, 2]
    fx, fy, cx, cy = intr
    with np.errstate(divide="ignore", invalid="ignore"):
        u = fx * xc[:, 0] / z + cx
        v = fy * xc[:, 1] / z + cy
    return np.stack([u, v], -1) - px, z, xc


def jacobian(xc, intr):
    fx, fy, _, _ = intr
    n = xc.shape[0]
    x, y, z = xc[:, 0], xc[:, 1], xc[:, 2]
    front = z > 0
    zs = np.where(front, z, 1.0)
    dpi = np.zeros((n, 2, 3))
    dpi[:, 0, 0] = fx / zs
    dpi[:, 0, 2] = -fx * x / (zs * zs)
    dpi[:, 1, 1] = fy / zs
    dpi[:, 1, 2] = -fy * y / (zs * zs)
    dx = np.zeros((n, 3, 6))
    dx[:, 0, 1], dx[:, 0, 2] = z, -y
    dx[:, 1, 0], dx[:, 1, 2] = -z, x
    dx[:, 2, 0], dx[:, 2, 1] = y, -x
    dx[:, 0, 3] = dx[:, 1, 4] = dx[:, 2, 5] = 1.0
    J = np.einsum("nij,njk->nik", dpi, dx)
    J[~front] = 0.0
    return J


def cost(pose, X, px, w, kind, scale, intr) -> float:
    r, z, _ = residuals(pose, X, px, intr)
    e2 = (r * r).sum(-1)
    front = z > 0
    b = _behind(kind, scale)
    if not front.all() and math.isinf(b):
        return math.inf
    return float(np.sum(w * np.where(front, _rho(kind, scale, np.where(front, e2, 0.0)), b)))


def refine(pose, X, px, w, kind, scale, intr, max_iters=100, gtol=1e-10, ctol=1e-12):
    """Returns (pose, converged, iterations, cost_trace)."""
    X = np.asarray(X, dtype=np.float64).reshape(-1, 3)
    px = np.asarray(px, dtype=np.float64).reshape(-1, 2)
    w = np.asarray(w, dtype=np.float64).reshape(-1)
    if X.shape[0] < 3:
        raise ValueError(f"refinement needs >= 3 matches, got {X.shape[0]}")
    c = cost(pose, X, px, w, kind, scale, intr)
    trace = [c]
    lam = 1e-6
    conv = False
    it = 0
    for it in range(1, max_iters + 1):
        r, z, xc = residuals(pose, X, px, intr)
        e2 = (r * r).sum(-1)
        front = z > 0
        wr = w * _wt(kind, scale, np.where(front, e2, np.inf)) * front
        J = jacobian(xc, intr)
        g = 2.0 * np.einsum("n,nki,nk->i", wr, J, r)
        if float(np.linalg.norm(g)) < gtol:
            conv = True
            break
        H = 2.0 * np.einsum("n,nki,nkj->ij", wr, J, J)
        dg = np.maximum(np.diag(H), 1e-12)
        ok = False
        for _ in range(25):
            try:
                step = np.linalg.solve(H + lam * np.diag(dg), -g)
            except np.linalg.LinAlgError:
                lam *= 10.0
                continue
            cand = apply_delta(pose, step)
            cc = cost(cand, X, px, w, kind, scale, intr)
            if cc <= c:
                ok = True
                break
            lam *= 10.0
            if lam > 1e14:
                break
        if not ok:
            break
        lam = max(lam / 3.0, 1e-12)
        drop = c - cc
        pose, c = cand, cc
        trace.append(c)
        if drop < ctol * max(c, 1e-300):
            conv = True
            break
    return pose, conv, it, trace
