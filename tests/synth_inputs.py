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


# ----------------------------------------------------------------------------- generator B
# Plane scene with analytic depth and bidirectional dense fields (BASELINE
# configs C2 / C5: 560^2 images, f = 280).  Written for this repo (the
# reference synth is not available on the GPU box); same shape of data as
# visloc.synth (plane patch, look-at cameras, corrupt() noise model).

def _look_at(center, target, roll):
    z = target - center
    z = z / np.linalg.norm(z)
    up = np.array([0.0, -1.0, 0.0])
    x = np.cross(up, z)
    x = x / np.linalg.norm(x)
    y = np.cross(z, x)
    Rc = np.stack([x, y, z])  # rows: camera axes in world
    cr, sr = math.cos(roll), math.sin(roll)
    Rr = np.array([[cr, -sr, 0.0], [sr, cr, 0.0], [0.0, 0.0, 1.0]])
    R = Rr @ Rc
    return R, -R @ center


class PlaneScene:
    def __init__(self, W=560, f=280.0, plane_z=3.0, extent=8.0, seed=0):
        self.W, self.f, self.c, self.plane_z, self.extent = W, f, W / 2.0, plane_z, extent
        self.rng = np.random.default_rng(seed)

    def camera(self, spread=0.3, backoff=0.25, roll_deg=3.0, rng=None):
        r = self.rng if rng is None else rng
        center = np.array([r.uniform(-spread, spread), r.uniform(-spread, spread),
                           -self.plane_z * backoff * r.uniform(0.0, 1.0)])
        return _look_at(center, np.array([0.0, 0.0, self.plane_z]), math.radians(r.uniform(-roll_deg, roll_deg)))

    def _hit(self, cam, u, v):
        R, t = cam
        d = np.stack([(u - self.c) / self.f, (v - self.c) / self.f, np.ones_like(u)], -1) @ R  # world dirs
        C = -R.T @ t
        s = (self.plane_z - C[2]) / d[..., 2]
        P = C + s[..., None] * d
        ok = (s > 0) & (np.abs(P[..., 0]) <= self.extent) & (np.abs(P[..., 1]) <= self.extent)
        return P, ok

    def depth_grid(self, cam, g):
        s = self.W / g
        u, v = np.meshgrid((np.arange(g) + 0.5) * s, (np.arange(g) + 0.5) * s)
        P, ok = self._hit(cam, u, v)
        z = (P @ cam[0].T + cam[1])[..., 2]
        ok &= z > 0
        return np.where(ok, z, 0.0).astype(np.float32), ok

    def field(self, cam_a, cam_b, g, rng, sigma=1.0, outlier_frac=0.7):
        """(targets (g,g,2) f32, conf (g,g) f32, scale): exact matches a->b, then corrupted."""
        s = self.W / g
        u, v = np.meshgrid((np.arange(g) + 0.5) * s, (np.arange(g) + 0.5) * s)
        P, ok = self._hit(cam_a, u, v)
        xc = P @ cam_b[0].T + cam_b[1]
        ok &= xc[..., 2] > 0
        with np.errstate(divide="ignore", invalid="ignore"):
            tu = self.f * xc[..., 0] / xc[..., 2] + self.c
            tv = self.f * xc[..., 1] / xc[..., 2] + self.c
        ok &= (tu >= 0) & (tu < self.W) & (tv >= 0) & (tv < self.W)
        tg = np.stack([tu, tv], -1) + rng.normal(0, sigma, (g, g, 2))
        conf = rng.uniform(0.5, 1.0, (g, g))
        out = ok & (rng.random((g, g)) < outlier_frac)
        tg[out] = rng.uniform(0, self.W, (int(out.sum()), 2))
        conf[out] = rng.uniform(0.0, 0.3, int(out.sum()))
        conf[~ok] = 0.0
        tg[~ok] = 0.0
        return tg.astype(np.float32), conf.astype(np.float32), s


def lifted_scene(K, Q, g, seed=0, depth_kind="f32", outlier_frac=0.7, sigma=1.0, only=None, fields="f64"):
    """(vmap, jobs, depth_cache) for the GPU package: K database cameras, Q query
    jobs with bidirectional fields to every database camera; depth as f32 / f16
    DepthMap (via the returned depth_cache) or u8 log codes (entry.qdepth).
    Each query draws from its own generator, so ``only=[i, ...]`` rebuilds a
    subset identically (CPU-baseline workers).  fields="f32" holds the fields
    as a file-backed (IMLC) field would: float32 targets and confidences."""
    from paper_2601_04185_b200.geometry import CameraIntrinsics, Pose, matrix_to_quat
    from paper_2601_04185_b200.localizer import (CorrespondenceField, DepthMap, FieldPair,
                                                 QuantizedDepthMap, QueryJob)
    sc = PlaneScene(seed=seed)
    intr = CameraIntrinsics(sc.f, sc.f, sc.c, sc.c, sc.W, sc.W)
    rng = np.random.default_rng(seed + 1)

    class Entry:
        pass

    class Map:
        pass

    entries, depth_cache = [], {}
    for k in range(K):
        cam = sc.camera()
        e = Entry()
        e.id = f"cam{k:03d}"
        e.pose = Pose(matrix_to_quat(cam[0]), cam[1])
        e.intrinsics = intr
        e.descriptor = rng.normal(size=16).astype(np.float32)
        e.cam = cam
        vals, valid = sc.depth_grid(cam, g)
        e.qdepth = None
        if depth_kind == "u8":
            span = math.log(128.0) - math.log(0.25)
            uq = (np.log(np.clip(vals.astype(np.float64), 0.25, 128.0)) - math.log(0.25)) / span
            codes = np.where(valid, 1 + np.floor(uq * 254 + 0.5), 0).astype(np.uint8)
            e.qdepth = QuantizedDepthMap(codes, 0.25, 128.0, 255, intr)
        else:
            dt = np.float16 if depth_kind == "f16" else np.float32
            depth_cache[e.id] = DepthMap(vals.astype(dt), valid, intr)
        entries.append(e)
    vmap = Map()
    vmap.entries = entries
    jobs = []
    for qi in (range(Q) if only is None else only):
        rng = np.random.default_rng([seed, 7, qi])
        cam = sc.camera(spread=0.24, rng=rng)
        fields = {}
        for e in entries:
            t1, c1, s = sc.field(cam, e.cam, g, rng, sigma, outlier_frac)
            t2, c2, _ = sc.field(e.cam, cam, g, rng, sigma, outlier_frac)
            if fields == "f32":
                t1, c1, t2, c2 = (a.astype(np.float32) for a in (t1, c1, t2, c2))
            fields[e.id] = FieldPair(query_to_db=CorrespondenceField("q", e.id, t1, c1, s, s),
                                     db_to_query=CorrespondenceField(e.id, "q", t2, c2, s, s))
        job = QueryJob(f"query{qi:04d}", intr, rng.normal(size=16), fields, k_loc=K)
        job.gt = Pose(matrix_to_quat(cam[0]), cam[1])
        jobs.append(job)
    return vmap, jobs, (depth_cache if depth_kind != "u8" else None)


def mapping_scene(E, V, g, seed=0, sigma=0.5, outlier_frac=0.3, only=None):
    """Mapping workload on the plane scene: E posed database images, entry i
    triangulated against the V next cameras (cyclic) with f32 fields i -> j.
    Returns [(entry, covisible, fields)] (``only`` selects entries; each entry's
    fields come from its own generator so subsets rebuild identically)."""
    from paper_2601_04185_b200.geometry import CameraIntrinsics, Pose, matrix_to_quat
    from paper_2601_04185_b200.matchio import CorrespondenceField
    sc = PlaneScene(seed=seed)
    intr = CameraIntrinsics(sc.f, sc.f, sc.c, sc.c, sc.W, sc.W)

    class Entry:
        pass

    ents = []
    for k in range(E):
        cam = sc.camera()
        e = Entry()
        e.id, e.cam, e.intrinsics = f"db{k:04d}", cam, intr
        e.pose = Pose(matrix_to_quat(cam[0]), cam[1])
        ents.append(e)
    jobs = []
    for i in (range(E) if only is None else only):
        rng = np.random.default_rng([seed, 11, i])
        covis = [ents[(i + 1 + k) % E] for k in range(V)]
        fields = []
        for c in covis:
            t, cf, s = sc.field(ents[i].cam, c.cam, g, rng, sigma, outlier_frac)
            fields.append(CorrespondenceField(ents[i].id, c.id, t, cf, s, s))
        jobs.append((ents[i], covis, fields))
    return jobs


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
