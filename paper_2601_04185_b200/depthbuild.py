"""Dense depth triangulation on the GPU — drop-in for ``visloc.depthbuild``.

SURVEY §8f row 3: the mapping step that produces the depth the lift consumes.
``build_depth_map`` / ``build_depth_maps`` triangulate every grid cell of one
or many database entries in one ``vl_build_depth_maps`` launch (a lane group
per pixel: gate + closest-point hypotheses, ballot voting, damped Newton on
the weighted squared angular error); ``triangulate_pixel`` /
``depth_hypothesis`` run explicit observation sets through
``vl_triangulate_rays``.  ``build_map_from_fields`` (mapbuild.py:36-81)
chains it with ``mapstore.quantize_depth_batch``: the whole map is
triangulated and quantised in two launches.

Reference: depthbuild.py:80-93 (TriangulationConfig), :104-189
(depth_hypothesis, triangulate_pixel), :230-246 (select_covisible), :249-375
(build_depth_map), :378-441 (refinement); mapbuild.py:36-81.  Checks and
their messages follow the reference (pairing, grid, span).  Inputs are
duck-typed: the reference's own entries / fields / poses work unchanged.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple, Sequence

import numpy as np

from . import _lib
from .geometry import CameraIntrinsics, Pose
from .localizer import DepthMap
from .retrieval import DescriptorIndex

__all__ = [
    "DepthBuildPlan", "DepthBuildReport", "DepthMap", "Observation", "TriangulationConfig", "build_depth_map", "build_depth_maps",
    "build_map_from_fields", "depth_hypothesis", "select_covisible", "triangulate_pixel",
]

MAX_VIEWS = 128  # covisible views per map / observations per problem on the device path


@dataclass(frozen=True)
class TriangulationConfig:
    angular_threshold_rad: float = math.radians(2.0)
    min_inliers: int = 4
    confidence_threshold: float = 0.05
    k_map: int = 50
    max_refine_iters: int = 20
    refine_tol: float = 1e-8

    def __post_init__(self) -> None:
        if self.angular_threshold_rad <= 0:
            raise ValueError("angular threshold must be positive")
        if self.min_inliers < 1:
            raise ValueError("min_inliers must be >= 1")


class Observation(NamedTuple):
    """A match against one covisible posed image."""

    pose: Pose
    intrinsics: CameraIntrinsics
    target_px: np.ndarray
    confidence: float


def _cfg_c(cfg) -> _lib.TriConfig:
    c = _lib.TriConfig()
    c.angular_threshold_rad = float(cfg.angular_threshold_rad)
    c.confidence_threshold = float(cfg.confidence_threshold)
    c.refine_tol = float(cfg.refine_tol)
    c.min_inliers = int(cfg.min_inliers)
    c.max_refine_iters = int(cfg.max_refine_iters)
    return c


def _fill_cam(rec, pose, intr):
    rt = np.asarray(pose.R, dtype=np.float64).T
    for i in range(9):
        rec.rt[i] = float(rt.flat[i])
    c = pose.center()
    for i in range(3):
        rec.center[i] = float(c[i])
    rec.fx, rec.fy, rec.cx, rec.cy = float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy)


# ----------------------------------------------------------------------------- explicit observation sets
def _solve_problems(problems, cfg, want_hyp=False):
    """problems: list of (ray, center, [Observation]) -> (depth (P,), count (P,), hyp list)."""
    import torch
    ctx = _lib.context()
    nobs = [len(p[2]) for p in problems]
    if max(nobs, default=0) > MAX_VIEWS:
        raise ValueError(f"at most {MAX_VIEWS} observations per pixel on the device path")
    tot = sum(nobs)
    P = (_lib.TriProblem * max(len(problems), 1))()
    O = (_lib.TriObs * max(tot, 1))()
    k = 0
    for i, (ray, center, obs) in enumerate(problems):
        r = np.asarray(ray, dtype=np.float64).reshape(3)
        c = np.asarray(center, dtype=np.float64).reshape(3)
        for j in range(3):
            P[i].ray[j], P[i].center[j] = float(r[j]), float(c[j])
        P[i].obs0, P[i].nobs = k, len(obs)
        for o in obs:
            _fill_cam(O[k], o.pose, o.intrinsics)
            px = np.asarray(o.target_px, dtype=np.float64).reshape(2)
            O[k].target[0], O[k].target[1] = float(px[0]), float(px[1])
            O[k].confidence = float(o.confidence)
            k += 1
    n = len(problems)
    dp = torch.from_numpy(np.frombuffer(bytes(P), dtype=np.uint8).copy()).cuda()
    do = torch.from_numpy(np.frombuffer(bytes(O), dtype=np.uint8).copy()).cuda()
    depth = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    count = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    hyp = torch.empty(max(tot, 1), dtype=torch.float64, device="cuda") if want_hyp else None
    rc = _lib.lib().vl_triangulate_rays(ctx.handle, dp.data_ptr(), n, do.data_ptr(), max(nobs, default=0),
                                        _lib.ctypes_ref(_cfg_c(cfg)), depth.data_ptr(), count.data_ptr(),
                                        hyp.data_ptr() if want_hyp else None, _lib.stream_ptr())
    ctx.check(rc, "vl_triangulate_rays")
    return depth.cpu().numpy()[:n], count.cpu().numpy()[:n], (hyp.cpu().numpy()[:tot] if want_hyp else None)


def depth_hypothesis(ref_ray, ref_center, obs: Observation):
    """Depth along the reference ray closest to the observation's ray, or None
    (parallel within 1e-12, or behind the reference camera; depthbuild.py:104-128)."""
    _, _, hyp = _solve_problems([(ref_ray, ref_center, [obs])], TriangulationConfig(), want_hyp=True)
    return None if not np.isfinite(hyp[0]) else float(hyp[0])


def triangulate_pixel(ref_ray, ref_center, observations: Sequence[Observation], cfg: TriangulationConfig):
    """(refined ray depth, winning inlier count) or None (depthbuild.py:151-189)."""
    if not observations:
        return None
    d, n, _ = _solve_problems([(ref_ray, ref_center, list(observations))], cfg)
    return None if n[0] == 0 else (float(d[0]), int(n[0]))


# ----------------------------------------------------------------------------- dense maps
def select_covisible(entry, vmap, k_map: int) -> list:
    """Top-``k_map`` entries by descriptor similarity excluding ``entry`` (depthbuild.py:230-246);
    host ranking identical to ``retrieval.DescriptorIndex.topk``."""
    index = DescriptorIndex.from_entries((e.id, e.descriptor) for e in vmap.entries if e.id != entry.id)
    if index.size == 0:
        return []
    ranked = index.topk(np.asarray(entry.descriptor, dtype=np.float64), k_map)
    by_id = {e.id: e for e in vmap.entries}
    return [by_id[eid] for eid, _ in ranked]


def _check_job(entry, covis, fields):
    """The reference's argument checks, in its order (depthbuild.py:262-286)."""
    if len(fields) != len(covis):
        raise ValueError(f"{len(fields)} fields for {len(covis)} covisible entries")
    if not fields:
        raise ValueError("need at least one correspondence field")
    intr = entry.intrinsics
    gh, gw = fields[0].grid_h, fields[0].grid_w
    for fld, cov in zip(fields, covis):
        if fld.source_id != entry.id or fld.target_id != cov.id:
            raise ValueError(f"field {fld.source_id}->{fld.target_id} does not pair {entry.id}->{cov.id}")
        if (fld.grid_h, fld.grid_w) != (gh, gw):
            raise ValueError("all fields must share one grid resolution")
        if abs(fld.grid_w * fld.scale_x - intr.width) > 1e-6 * intr.width or \
           abs(fld.grid_h * fld.scale_y - intr.height) > 1e-6 * intr.height:
            raise ValueError(f"field grid for {entry.id} does not span the image "
                             f"({fld.grid_w}x{fld.grid_h} at scale {fld.scale_x}x{fld.scale_y})")
    if len(fields) > MAX_VIEWS:
        raise ValueError(f"at most {MAX_VIEWS} covisible views per map on the device path")
    return gh, gw


_VIEW_DTYPE = np.dtype([("targets", "<u8"), ("confidence", "<u8"), ("rt", "<f8", 9), ("center", "<f8", 3),
                        ("fx", "<f8"), ("fy", "<f8"), ("cx", "<f8"), ("cy", "<f8")])          # vl_tri_view
_MAP_DTYPE = np.dtype([("grid_w", "<i4"), ("grid_h", "<i4"), ("view0", "<i4"), ("nview", "<i4"),
                       ("fx", "<f8"), ("fy", "<f8"), ("cx", "<f8"), ("cy", "<f8"), ("sx", "<f8"), ("sy", "<f8"),
                       ("R", "<f8", 9), ("center", "<f8", 3), ("depth", "<u8"), ("valid", "<u8")])  # vl_tri_map
assert _VIEW_DTYPE.itemsize == 144 and _MAP_DTYPE.itemsize == 176


class _Staging:
    """Pinned host staging buffers reused across plans (a pinned allocation
    costs tens of ms); a buffer is refilled only after its H2D has completed."""

    def __init__(self):
        self.bufs = []  # [tensor, event or None]

    def get(self, nbytes: int):
        import torch
        for b in self.bufs:
            if b[0].numel() >= nbytes and (b[1] is None or b[1].query()):
                return b
        b = [torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True), None]
        self.bufs.append(b)
        if len(self.bufs) > 4:
            self.bufs = [x for x in self.bufs[:-4] if x[1] is not None and not x[1].query()] + self.bufs[-4:]
        return b


_STAGING = _Staging()


def _cam_record(pose, intr, cache):
    """(R^T row-major, centre, fx, fy, cx, cy) of a camera, computed once per pose object."""
    key = id(pose)
    r = cache.get(key)
    if r is None:
        r = (np.asarray(pose.R, dtype=np.float64).T.reshape(-1), np.asarray(pose.center(), dtype=np.float64),
             float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy), pose)
        cache[key] = r
    return r


def _pack_planar(fields, host, dt, tot_cells, c_off):
    """Targets (2 values / cell) then confidences into the pinned buffer,
    field ranges split over a few threads (numpy copies release the GIL;
    one thread copies ~5 GB/s).  VISLOC_PACK_THREADS overrides the count."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    n = len(fields)
    nt = int(os.environ.get("VISLOC_PACK_THREADS", 0)) or min(4, max(1, (os.cpu_count() or 1) // 2))
    nt = max(1, min(nt, n // 32 or 1))

    def work(lo, hi):
        a, b = int(c_off[lo]), int(c_off[hi])
        np.concatenate([np.asarray(f.targets, dtype=dt).reshape(-1) for f in fields[lo:hi]], out=host[2 * a:2 * b])
        np.concatenate([np.asarray(f.confidence, dtype=dt).reshape(-1) for f in fields[lo:hi]],
                       out=host[2 * tot_cells + a:2 * tot_cells + b])
    if nt == 1:
        work(0, n)
        return
    cuts = [n * k // nt for k in range(nt + 1)]
    with ThreadPoolExecutor(nt) as ex:
        for f in [ex.submit(work, cuts[k], cuts[k + 1]) for k in range(nt)]:
            f.result()


class DepthBuildPlan:
    """Many entries' fields resident in HBM, ready to triangulate (the device-resident path).

    Construction does the host work once (checks, field packing into a pooled
    pinned buffer + one H2D, map / view records as numpy structured arrays
    with per-camera values computed once per pose); ``run()`` launches
    ``vl_build_depth_maps`` into the plan's device outputs ``depth`` (f32) /
    ``valid`` (u8), packed map after map."""

    def __init__(self, jobs, cfg: TriangulationConfig):
        import torch
        self.jobs = list(jobs)
        self.cfg = cfg
        self.shapes = [_check_job(*j) for j in self.jobs]
        _lib.context()
        fields = [f for _, _, fl in self.jobs for f in fl]
        self.f64 = any(np.asarray(f.confidence).dtype != np.float32 or np.asarray(f.targets).dtype != np.float32
                       for f in fields)
        dt = np.dtype(np.float64 if self.f64 else np.float32)
        item = dt.itemsize
        ncell = np.fromiter((f.grid_w * f.grid_h for f in fields), dtype=np.int64, count=len(fields))
        c_off = np.concatenate([[0], np.cumsum(ncell)]).astype(np.int64)
        tot_cells = int(c_off[-1])
        # one pinned buffer: targets (2 values / cell) then confidences (1 / cell)
        nbytes = 3 * tot_cells * item
        stage = _STAGING.get(nbytes)
        host = stage[0].numpy()[:nbytes].view(dt)
        if fields:
            _pack_planar(fields, host, dt, tot_cells, c_off)
        self.D = torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")
        self.D[:nbytes].copy_(stage[0][:nbytes], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        stage[1] = ev
        self.field_bytes = nbytes
        base = self.D.data_ptr()
        self.npix = [h * w for h, w in self.shapes]
        self.p_off = np.concatenate([[0], np.cumsum(self.npix)]).astype(np.int64)
        tot = max(int(self.p_off[-1]), 1)
        self.depth = torch.empty(tot, dtype=torch.float32, device="cuda")
        self.valid = torch.empty(tot, dtype=torch.uint8, device="cuda")
        self.nviews = len(fields)
        views = np.zeros(max(len(fields), 1), dtype=_VIEW_DTYPE)
        maps = np.zeros(max(len(self.jobs), 1), dtype=_MAP_DTYPE)
        if fields:
            views["targets"][:len(fields)] = base + 2 * c_off[:-1] * item
            views["confidence"][:len(fields)] = base + (2 * tot_cells + c_off[:-1]) * item
        cache = {}
        cams = [_cam_record(cov.pose, cov.intrinsics, cache) for _, covis, _ in self.jobs for cov in covis]
        if cams:
            views["rt"][:len(cams)] = np.stack([c[0] for c in cams])
            views["center"][:len(cams)] = np.stack([c[1] for c in cams])
            for k, name in enumerate(("fx", "fy", "cx", "cy")):
                views[name][:len(cams)] = [c[2 + k] for c in cams]
        v = 0
        for m, ((entry, covis, fl), (gh, gw)) in enumerate(zip(self.jobs, self.shapes)):
            M = maps[m]
            intr = entry.intrinsics
            M["grid_w"], M["grid_h"], M["view0"], M["nview"] = gw, gh, v, len(fl)
            M["fx"], M["fy"], M["cx"], M["cy"] = float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy)
            M["sx"], M["sy"] = intr.width / gw, intr.height / gh
            M["R"] = np.asarray(entry.pose.R, dtype=np.float64).reshape(-1)
            M["center"] = np.asarray(entry.pose.center(), dtype=np.float64)
            M["depth"] = self.depth.data_ptr() + int(self.p_off[m]) * 4
            M["valid"] = self.valid.data_ptr() + int(self.p_off[m])
            v += len(fl)
        self._views, self._maps = views, maps  # kept alive: the C call reads them
        self._cfg = _cfg_c(cfg)

    @property
    def pixels(self) -> int:
        return int(self.p_off[-1])

    def run(self):
        ctx = _lib.context()
        if not self.jobs:
            return self
        import ctypes as C
        rc = _lib.lib().vl_build_depth_maps(ctx.handle, self._maps.ctypes.data_as(C.POINTER(_lib.TriMap)),
                                            len(self.jobs), self._views.ctypes.data_as(C.POINTER(_lib.TriView)),
                                            self.nviews, 1 if self.f64 else 0, _lib.ctypes_ref(self._cfg),
                                            _lib.stream_ptr())
        ctx.check(rc, "vl_build_depth_maps")
        return self

    def device_maps(self):
        """[(depth (gh,gw) f32, valid (gh,gw) u8)] CUDA tensor views of the outputs."""
        out = []
        for m, (gh, gw) in enumerate(self.shapes):
            sl = slice(int(self.p_off[m]), int(self.p_off[m + 1]))
            out.append((self.depth[sl].view(gh, gw), self.valid[sl].view(gh, gw)))
        return out

    def host_maps(self) -> list:
        dh, vh = self.depth.cpu().numpy(), self.valid.cpu().numpy().astype(bool)
        out = []
        for m, ((entry, _, _), (gh, gw)) in enumerate(zip(self.jobs, self.shapes)):
            sl = slice(int(self.p_off[m]), int(self.p_off[m + 1]))
            out.append(DepthMap(values=dh[sl].reshape(gh, gw).copy(), valid=vh[sl].reshape(gh, gw).copy(),
                                intrinsics=entry.intrinsics))
        return out


def build_depth_maps(jobs, cfg: TriangulationConfig, device_out: bool = False) -> list:
    """``build_depth_map`` of many entries in one launch.

    ``jobs``: sequence of (entry, covisible_entries, fields).  Returns
    DepthMaps (host arrays), or (depth f32, valid u8) CUDA tensor pairs with
    ``device_out=True``."""
    plan = DepthBuildPlan(jobs, cfg).run()
    return plan.device_maps() if device_out else plan.host_maps()


def build_depth_map(entry, covisible_entries: Sequence, fields: Sequence, cfg: TriangulationConfig,
                    chunk_pixels: int = 4096) -> DepthMap:
    """Drop-in ``depthbuild.build_depth_map`` (depthbuild.py:249-375).  ``chunk_pixels`` is
    accepted for signature compatibility; the output never depends on it."""
    return build_depth_maps([(entry, list(covisible_entries), list(fields))], cfg)[0]


# ----------------------------------------------------------------------------- mapbuild
@dataclass
class DepthBuildReport:
    entry_id: str
    valid_fraction: float
    num_covisible: int
    depth: object = None


def build_map_from_fields(posed_entries, fields_lookup, cfg: TriangulationConfig, d_min: float = 0.25,
                          d_max: float = 128.0, levels: int = 255):
    """Drop-in ``mapbuild.build_map_from_fields`` (mapbuild.py:36-81): covisibility on the host
    (reference-exact ranking), every entry triangulated in one launch and quantised in one."""
    from .mapstore import Map, MapEntry, quantize_depth_batch
    mod = type(posed_entries[0]).__module__ if posed_entries else ""
    if mod.startswith("visloc."):  # build the reference's own container types
        import importlib
        ms = importlib.import_module("visloc.mapstore")
        Map, MapEntry = ms.Map, ms.MapEntry
    vmap = Map(entries=list(posed_entries))
    jobs = []
    for entry in posed_entries:
        covis = select_covisible(entry, vmap, cfg.k_map)
        jobs.append((entry, covis, [fields_lookup(entry, c) for c in covis]))
    depths = build_depth_maps(jobs, cfg)
    qds = quantize_depth_batch(depths, d_min, d_max, levels)
    out, reports = [], []
    for (entry, covis, _), depth, qd in zip(jobs, depths, qds):
        out.append(MapEntry(id=entry.id, pose=entry.pose, intrinsics=entry.intrinsics,
                            rgb_payload=entry.rgb_payload, rgb_codec=entry.rgb_codec, qdepth=qd,
                            descriptor=entry.descriptor))
        reports.append(DepthBuildReport(entry_id=entry.id, valid_fraction=float(depth.valid.mean()),
                                        num_covisible=len(covis), depth=depth))
    return Map(entries=out, rgb_codec=vmap.rgb_codec), reports
