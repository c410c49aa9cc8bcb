"""MSAC scoring and the LO-RANSAC driver restated from the reference.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``pkg/src/visloc/posest.py``:

* ``required_iterations`` :106-120 — ceil(ln eta / log1p(-eps^3)), clamped;
* ``errors_sq`` / ``msac`` :137-175 — fp64, behind-camera -> +inf error,
  cost sum w min(e2, tau^2), flags e2 < tau^2;
* ``score_fp32`` :178-220 — the fp32 ranking cost of every hypothesis;
* ``ransac`` :223-299 — stride subset (<= max_scoring), batches of seeded
  3-samples (``oracle.rng``), P3P, fp32 scores, ordered first-better scan
  with LM local optimisation on every new best, adaptive stop on the subset
  inlier ratio, fp64 full-set classification and Cauchy final refinement;
* bearings :302-311.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .geometry import canon, pose_from_Rt, q2R
from .p3p import p3p_batch
from .refine import CAUCHY, TRUNCATED, refine
from .rng import PCG64Stream

SCORE_CHUNK = 256


def required_iterations(eps, eta, m=3, cap=100_000) -> int:
    eps = min(max(eps, 0.0), 1.0)
    if eps <= 0.0:
        return cap
    if eps >= 1.0:
        return 1
    den = math.log1p(-(eps ** m))
    if den == 0.0:
        return cap
    return int(min(max(math.ceil(math.log(eta) / den), 1), cap))


def errors_sq(R, t, X, px, intr):
    fx, fy, cx, cy = intr
    xc = X @ R.T
    xc += t
    z = xc[:, 2]
    front = z > 0
    zs = np.where(front, z, 1.0)
    du = fx * xc[:, 0]
    du /= zs
    du += cx - px[:, 0]
    dv = fy * xc[:, 1]
    dv /= zs
    dv += cy - px[:, 1]
    e2 = du * du
    e2 += dv * dv
    return np.where(front, e2, np.inf)


def msac(pose, px, X, w, intr, tau):
    e2 = errors_sq(q2R(pose[0]), pose[1], X, px, intr)
    t2 = tau * tau
    return float(np.einsum("n,n->", w, np.minimum(e2, t2))), e2 < t2


def score_fp32(Rs, ts, X, px, w, intr, tau):
    fx, fy, cx, cy = intr
    nh, n = Rs.shape[0], X.shape[0]
    X32 = np.ascontiguousarray(X, dtype=np.float32)
    t2 = np.float32(tau * tau)
    out = np.empty(nh, dtype=np.float64)
    uo = (cx - px[:, 0][:, None]).astype(np.float32)
    vo = (cy - px[:, 1][:, None]).astype(np.float32)
    w32 = w.astype(np.float32)
    f32x, f32y = np.float32(fx), np.float32(fy)
    for a in range(0, nh, SCORE_CHUNK):
        b = min(a + SCORE_CHUNK, nh)
        h = b - a
        xc = X32 @ Rs[a:b].reshape(3 * h, 3).T.astype(np.float32)
        xc += ts[a:b].reshape(1, 3 * h).astype(np.float32)
        xc = xc.reshape(n, h, 3)
        z = xc[:, :, 2]
        front = z > 0
        zs = np.where(front, z, np.float32(1.0))
        du = f32x * xc[:, :, 0]
        du /= zs
        du += uo
        dv = f32y * xc[:, :, 1]
        dv /= zs
        dv += vo
        e2 = du * du
        e2 += dv * dv
        np.minimum(e2, t2, out=e2)
        e2[~front] = t2
        out[a:b] = np.einsum("n,nh->h", w32, e2)
    return out


def bearings(px, intr):
    fx, fy, cx, cy = intr
    b = np.stack([(px[:, 0] - cx) / fx, (px[:, 1] - cy) / fy, np.ones(px.shape[0])], -1)
    return b / np.linalg.norm(b, axis=-1, keepdims=True)


@dataclass
class Config:
    max_iterations: int = 100_000
    batch_size: int = 1_000
    miss_probability: float = 1e-4
    reproj_threshold: float = 12.0
    max_scoring: int = 10_000
    cauchy_scale: float | None = None
    lm_max_iters: int = 100
    seed: int = 0

    @property
    def cauchy(self):
        return self.reproj_threshold if self.cauchy_scale is None else self.cauchy_scale


@dataclass
class Result:
    q: np.ndarray
    t: np.ndarray
    inlier_count: int
    inlier_flags: np.ndarray
    score: float
    iterations: int
    converged: bool
    lo_calls: int = 0
    hypotheses: int = 0
    evals: int = 0
    trace: dict = field(default_factory=dict)


def ransac(px, X, w, intr, cfg: Config, keep_trace=False) -> Result:
    """``ransac_pnp`` restated; ``intr`` = (fx, fy, cx, cy)."""
    px = np.asarray(px, dtype=np.float64).reshape(-1, 2)
    X = np.asarray(X, dtype=np.float64).reshape(-1, 3)
    w = np.asarray(w, dtype=np.float64).reshape(-1)
    n = px.shape[0]
    if n < 3:
        raise ValueError(f"need >= 3 matches, got {n}")
    stride = math.ceil(n / cfg.max_scoring)
    pxs, Xs, ws = px[::stride], X[::stride], w[::stride]
    nsub = pxs.shape[0]
    tau = cfg.reproj_threshold
    gen = PCG64Stream.from_seed(cfg.seed)
    bear = bearings(px, intr)
    best = None
    best_cost = math.inf
    iters = 0
    lo_calls = hyps = evals = 0
    tr = {"samples": [], "nhyp": [], "costs": [], "lo": []} if keep_trace else {}
    while iters < cfg.max_iterations:
        bn = min(cfg.batch_size, cfg.max_iterations - iters)
        samp = np.array([gen.choice3(n) for _ in range(bn)], dtype=np.int64)
        Rs, ts, _ = p3p_batch(bear[samp], X[samp])
        iters += bn
        if keep_trace:
            tr["samples"].append(samp)
            tr["nhyp"].append(Rs.shape[0])
        if Rs.shape[0] > 0:
            costs = score_fp32(Rs, ts, Xs, pxs, ws, intr, tau)
            hyps += Rs.shape[0]
            evals += Rs.shape[0] * nsub
            if keep_trace:
                tr["costs"].append(costs)
            for h in range(costs.shape[0]):
                if costs[h] < best_cost:
                    best_cost = float(costs[h])
                    best = pose_from_Rt(Rs[h], ts[h])
                    lo_pose, _, _, _ = refine(best, Xs, pxs, ws, TRUNCATED, tau, intr,
                                              max_iters=cfg.lm_max_iters)
                    lo_calls += 1
                    lo_cost, _ = msac(lo_pose, pxs, Xs, ws, intr, tau)
                    if keep_trace:
                        tr["lo"].append((len(tr["costs"]) - 1, h, best_cost, lo_cost))
                    if lo_cost < best_cost:
                        best_cost = lo_cost
                        best = lo_pose
        if best is not None:
            _, sf = msac(best, pxs, Xs, ws, intr, tau)
            need = required_iterations(int(sf.sum()) / nsub, cfg.miss_probability, 3,
                                       cfg.max_iterations)
            if iters >= need:
                break
    common = dict(iterations=iters, lo_calls=lo_calls, hypotheses=hyps, evals=evals, trace=tr)
    if best is None:
        return Result(np.array([1.0, 0, 0, 0]), np.zeros(3), 0, np.zeros(n, dtype=bool),
                      math.inf, converged=False, **common)
    c_full, f_full = msac(best, px, X, w, intr, tau)
    if int(f_full.sum()) < 3:
        return Result(best[0], best[1], int(f_full.sum()), f_full, c_full,
                      converged=False, **common)
    fin, _, _, _ = refine(best, X[f_full], px[f_full], w[f_full], CAUCHY, cfg.cauchy, intr,
                          max_iters=cfg.lm_max_iters)
    sc, fl = msac(fin, px, X, w, intr, tau)
    return Result(fin[0], fin[1], int(fl.sum()), fl, sc, converged=True, **common)


__all__ = ["Config", "Result", "bearings", "canon", "errors_sq", "msac", "ransac",
           "required_iterations", "score_fp32"]
