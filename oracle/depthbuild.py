"""Dense depth triangulation restated from the reference (numpy, fp64) — TEST INFRASTRUCTURE ONLY.

Follows ``pkg/src/visloc/depthbuild.py``: ``build_depth_map`` :249-375 (gate,
world bearings, closest-point hypotheses, angular voting with first-maximum
winner, min-inlier gate) and the vectorised damped Newton
``_refine_depth_vec`` :408-441 with ``_vec_cost`` :378-384 and
``_vec_gradient`` :387-405.  Inputs are plain arrays (fields stacked per view,
poses as R / centre) so the GPU box can replay golden scenes.  Pinned bit for
bit to ``tests/golden/depthbuild.npz`` (made by the real reference).
"""

from __future__ import annotations

import numpy as np

PARALLEL_TOL = 1e-12


def _angles(points, centers, bearings):
    """Angle between (point - centre) and the observed bearing, per view."""
    rel = points - centers
    s = np.linalg.norm(np.cross(rel, bearings), axis=-1)
    return np.arctan2(s, np.sum(rel * bearings, axis=-1))


def _cost(d, rays, c_ref, centers, bearings, weights):
    ang = _angles((c_ref + d[:, None] * rays)[:, None, :], centers[None], bearings)
    return np.sum(weights * ang * ang, axis=-1)


def _grad(d, rays, c_ref, centers, bearings, weights):
    rel = (c_ref + d[:, None] * rays)[:, None, :] - centers[None]
    cr = np.cross(rel, bearings)
    s = np.linalg.norm(cr, axis=-1)
    c = np.sum(rel * bearings, axis=-1)
    theta = np.arctan2(s, c)
    rb = np.cross(rays[:, None, :], bearings)
    with np.errstate(divide="ignore", invalid="ignore"):
        ds = np.where(s > 0, np.sum(cr * rb, axis=-1) / np.where(s > 0, s, 1.0), 0.0)
        dc = np.sum(bearings * rays[:, None, :], axis=-1)
        n2 = s * s + c * c
        dth = np.where(n2 > 0, (ds * c - s * dc) / np.where(n2 > 0, n2, 1.0), 0.0)
    return np.sum(2.0 * weights * theta * dth, axis=-1)


def _newton(d, rays, c_ref, centers, bearings, weights, active, max_iters, tol):
    d = d.astype(np.float64).copy()
    active = active.copy()
    cost = _cost(d, rays, c_ref, centers, bearings, weights)
    for _ in range(max_iters):
        if not active.any():
            break
        g = _grad(d, rays, c_ref, centers, bearings, weights)
        h = np.maximum(1e-7 * np.abs(d), 1e-10)
        hess = (_grad(d + h, rays, c_ref, centers, bearings, weights)
                - _grad(d - h, rays, c_ref, centers, bearings, weights)) / (2.0 * h)
        newton = (hess > 0) & np.isfinite(hess) & np.isfinite(g)
        step = np.where(newton, -g / np.where(newton, hess, 1.0), -np.sign(g) * 0.05 * np.abs(d))
        step = np.where(active, step, 0.0)
        done = np.zeros_like(active)
        new_cost = cost.copy()
        for _ in range(30):
            trying = active & ~done
            if not trying.any():
                break
            cand = d + step
            pos = cand > 0
            cc = _cost(np.where(pos, cand, d), rays, c_ref, centers, bearings, weights)
            ok = trying & pos & (cc <= cost)
            new_cost = np.where(ok, cc, new_cost)
            done |= ok
            step = np.where(trying & ~ok, step * 0.5, step)
        conv = done & (np.abs(step) < tol * np.maximum(np.abs(d), 1e-300))
        d = np.where(done, d + step, d)
        cost = np.where(done, new_cost, cost)
        active &= done & ~conv
    return d


def build_depth_map(targets, conf, scale, ref_R, ref_C, ref_intr, view_R, view_C, view_intr, thr, min_inliers,
                    conf_thr, max_iters, tol):
    """targets (V,gh,gw,2), conf (V,gh,gw); ref_intr / view_intr rows (fx, fy, cx, cy, W, H);
    view_R (V,3,3) camera-from-world; returns (depth f32 (gh,gw), valid bool)."""
    V, gh, gw = conf.shape
    P = gh * gw
    cf = conf.reshape(V, P).T.astype(np.float64)                      # (P, V)
    tg = targets.reshape(V, P, 2).transpose(1, 0, 2).astype(np.float64)
    ok = (cf >= conf_thr) & (cf > 0)
    vi = np.asarray(view_intr, dtype=np.float64)
    with np.errstate(invalid="ignore"):
        bx = (tg[..., 0] - vi[:, 2]) / vi[:, 0]
        by = (tg[..., 1] - vi[:, 3]) / vi[:, 1]
        bc = np.stack([bx, by, np.ones_like(bx)], axis=-1)
        bc /= np.linalg.norm(bc, axis=-1, keepdims=True)
        bear = np.einsum("vij,pvj->pvi", np.ascontiguousarray(np.transpose(view_R, (0, 2, 1))), bc)
    bear = np.where(ok[..., None], bear, 0.0)
    fx, fy, cx, cy, W, H = ref_intr
    cols, rows = np.meshgrid(np.arange(gw), np.arange(gh))
    u = (cols + 0.5).reshape(-1) * (W / gw)
    v = (rows + 0.5).reshape(-1) * (H / gh)
    k = np.stack([(u - cx) / fx, (v - cy) / fy, np.ones(P)], axis=-1)
    kn = np.linalg.norm(k, axis=-1)
    k /= kn[:, None]
    rays = k @ np.asarray(ref_R).T.T
    wv = view_C - ref_C
    beta = np.einsum("pvd,pd->pv", bear, rays)
    den = 1.0 - beta * beta
    with np.errstate(divide="ignore", invalid="ignore"):
        D = (rays @ wv.T - beta * np.einsum("pvd,vd->pv", bear, wv)) / den
    hyp = ok & (den >= PARALLEL_TOL) & np.isfinite(D) & (D > 0)
    # votes[p, j, v]: view v agrees with hypothesis j of pixel p
    X = ref_C + D[..., None] * rays[:, None, :]
    rel = X[:, :, None, :] - view_C[None, None]
    ang = np.arctan2(np.linalg.norm(np.cross(rel, bear[:, None]), axis=-1), np.sum(rel * bear[:, None], axis=-1))
    votes = (ang < thr) & ok[:, None, :] & hyp[:, :, None]
    counts = votes.sum(axis=-1)
    j = np.argmax(counts, axis=1)
    idx = np.arange(P)
    keep = counts[idx, j] >= min_inliers
    depth = np.zeros(P)
    valid = np.zeros(P, dtype=bool)
    if keep.any():
        w = np.where(votes[idx, j, :] & keep[:, None], cf, 0.0)
        d = _newton(np.where(keep, D[idx, j], 1.0), rays, ref_C, view_C, bear, w, keep, max_iters, tol)
        depth[keep] = d[keep] / kn[keep]
        valid[keep] = True
    return np.where(valid, depth, 0.0).astype(np.float32).reshape(gh, gw), valid.reshape(gh, gw)
