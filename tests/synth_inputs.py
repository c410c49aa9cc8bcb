"""Seeded synthetic inputs shared by golden generation, tests and bench.

Generator A follows the reference test model ``pkg/tests/test_posest.py:18-35``
(intrinsics fx=fy=700, c=350; GT rotvec (0.05,-0.1,0.2), t=(0.1,0.2,0.3);
camera-frame points x,y~U(-1.2,1.2), z~U(2,5); outliers uniform in the
image with low weights).  ``refine_problem`` follows ``test_refine.py:22-33``.
Pure numpy — usable on the GPU box where the reference is absent.
"""

from __future__ import annotations

import math

import numpy as np


class _Intr:
    def __init__(self, fx, fy, cx, cy, width, height):
        self.fx, self.fy, self.cx, self.cy, self.width, self.height = fx, fy, cx, cy, width, height


def _rotvec_R(w):
    w = np.asarray(w, dtype=np.float64)
    th = np.linalg.norm(w)
    if th < 1e-15:
        return np.eye(3)
    k = w / th
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + math.sin(th) * K + (1 - math.cos(th)) * K @ K


try:  # the reference types when available (golden generation), else light stand-ins
    from visloc.geometry import CameraIntrinsics as _CI, Pose as _P, rotvec_to_quat as _r2q
    INTR_A = _CI(700.0, 700.0, 350.0, 350.0, 700, 700)
    GT_A = _P(_r2q(np.array([0.05, -0.1, 0.2])), np.array([0.1, 0.2, 0.3]))
    _GT_R, _GT_t = GT_A.R, GT_A.t
except Exception:  # pragma: no cover - GPU box / no reference
    INTR_A = _Intr(700.0, 700.0, 350.0, 350.0, 700, 700)
    GT_A = None
    _GT_R, _GT_t = None, np.array([0.1, 0.2, 0.3])


def gt_a():
    """(R, t) of the generator-A ground truth, computed like the reference Pose."""
    from oracle.geometry import q2R, rotvec2q, canon
    q = canon(rotvec2q(np.array([0.05, -0.1, 0.2])))
    return q, q2R(q), np.array([0.1, 0.2, 0.3])


def matches_a(n, outlier_frac=0.0, sigma=0.0, seed=0, R=None, t=None):
    """(px, X, w, outliers) exactly like test_posest._matches (test_posest.py:22-35)."""
    if R is None:
        _, R, t = gt_a()
    rng = np.random.default_rng(seed)
    xc = np.stack([rng.uniform(-1.2, 1.2, n), rng.uniform(-1.2, 1.2, n), rng.uniform(2.0, 5.0, n)], -1)
    xw = (xc - t) @ R
    z = xc[:, 2]
    px = np.stack([700.0 * xc[:, 0] / z + 350.0, 700.0 * xc[:, 1] / z + 350.0], -1)
    w = rng.uniform(0.5, 1.0, n)
    out = rng.random(n) < outlier_frac
    px = px + rng.normal(0, 1.0, (n, 2)) * sigma
    px[out] = rng.uniform(0, 700, (int(out.sum()), 2))
    w[out] = rng.uniform(0.05, 0.3, int(out.sum()))
    return px, xw, w, out


def random_pose(rng, rot_scale=0.3, t_scale=0.3):
    from oracle.geometry import canon, q2R, rotvec2q
    q = canon(rotvec2q(rng.normal(size=3) * rot_scale))
    return q, q2R(q), rng.normal(size=3) * t_scale


def refine_problem(rng, n, noise, outlier_frac):
    """Start pose perturbed from GT, points, pixels, weights (test_refine.py:22-33 style)."""
    from oracle.geometry import canon, qmul, rotvec2q
    q, R, t = random_pose(rng)
    xc = np.stack([rng.uniform(-1.2, 1.2, n), rng.uniform(-1.0, 1.0, n), rng.uniform(2.0, 6.0, n)], -1)
    X = (xc - t) @ R
    px = np.stack([700.0 * xc[:, 0] / xc[:, 2] + 350.0, 700.0 * xc[:, 1] / xc[:, 2] + 350.0], -1)
    px = px + rng.normal(0, noise, px.shape)
    out = rng.random(n) < outlier_frac
    px[out] = rng.uniform(0, 700, (int(out.sum()), 2))
    w = rng.uniform(0.3, 1.0, n)
    dq = rotvec2q(rng.normal(size=3) * 0.005)
    q0 = canon(qmul(dq, q))
    t0 = t + rng.normal(size=3) * 0.02
    try:
        from visloc.geometry import Pose as _P
        start = _P(q0, t0)
    except Exception:  # pragma: no cover
        start = (q0, t0)
    return start, X, px, w


def batch_a(Q, n, outlier_frac, sigma, seed0):
    """Q generator-A queries with per-query random GT poses (bench C1/C3/C4 inputs)."""
    pxs, Xs, ws = [], [], []
    for qi in range(Q):
        rng = np.random.default_rng(seed0 + qi)
        _, R, t = random_pose(rng, 0.2, 0.2)
        px, X, w, _ = matches_a(n, outlier_frac, sigma, seed=seed0 + 7919 * qi + 1, R=R, t=t)
        pxs.append(px)
        Xs.append(X)
        ws.append(w)
    return pxs, Xs, ws
