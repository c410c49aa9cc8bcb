"""Query-time lifting and localisation — drop-in for ``visloc.localizer``.

``lift`` / ``lift_arrays`` / ``localize`` / ``localize_batch`` run the
confidence gate, depth decode (f32, f16 or log-quantised codes), depth fetch
(direct or bilinear with the all-4-valid rule), unprojection and world
transform on the GPU (``vl_lift``), then feed the device-resident matches
straight into the batched estimator (``vl_ransac_pnp``).

Reference: ``localizer.py`` — ``interp_depth_many`` :87-115, ``lift``
:134-197, ``localize`` :200-238; ``matchio.filter_matches_arrays``
:203-218; ``mapstore.dequantize_depth`` :122-134.  Inputs are duck-typed so
the reference's own ``QueryJob`` / ``FieldPair`` / ``CorrespondenceField`` /
``DepthMap`` / ``QuantizedDepthMap`` / ``MapEntry`` objects work unchanged.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .geometry import CameraIntrinsics, Pose, pose_error
from .matchio import CorrespondenceField, FieldBlob, filter_matches_arrays  # noqa: F401
from .retrieval import DescriptorIndex
from .posest import (Match2D3D, PoseEstimate, RansacConfig, _estimates_from, _estimates_from_host, _stage_results,
                     ransac_pnp_device)

__all__ = [
    "CONFIDENCE_THRESHOLD", "CorrespondenceField", "DepthMap", "DescriptorIndex", 
    "FieldPair",
    "QuantizedDepthMap", "QueryJob", "dequantize_depth", "filter_matches_arrays", "interp_depth",
    "interp_depth_many", "LiftPlan", "lift", "lift_arrays", "localize", "localize_batch", "localize_pipelined",
    "serving_schedule",
]

CONFIDENCE_THRESHOLD = 0.05
DEFAULT_D_MIN = 0.25
DEFAULT_D_MAX = 128.0

KIND_F32, KIND_F16, KIND_CODE8, KIND_CODE16 = 0, 1, 2, 3


# ----------------------------------------------------------------------------- types
@dataclass
class DepthMap:
    """z-depth (f32) + validity at match-grid resolution (depthbuild.py:45-77)."""

    values: np.ndarray
    valid: np.ndarray
    intrinsics: CameraIntrinsics

    def __post_init__(self):
        # float16 storage is kept as-is (compressed-map HBM format); every f16
        # value widens exactly to the f32 the reference would hold
        half = np.asarray(self.values).dtype == np.float16
        self.values = np.ascontiguousarray(self.values, dtype=np.float16 if half else np.float32)
        self.valid = np.ascontiguousarray(self.valid, dtype=bool)
        if self.values.shape != self.valid.shape or self.values.ndim != 2:
            raise ValueError("values and valid must be equal 2-D shapes")
        if np.any(self.valid & ~(np.isfinite(self.values) & (self.values > 0))):
            raise ValueError("valid pixels must hold positive finite depth")

    @property
    def height(self) -> int:
        return self.values.shape[0]

    @property
    def width(self) -> int:
        return self.values.shape[1]


@dataclass
class QuantizedDepthMap:
    """Log-space depth codes; 0 invalid (mapstore.py:65-93)."""

    codes: np.ndarray
    d_min: float = DEFAULT_D_MIN
    d_max: float = DEFAULT_D_MAX
    levels: int = 255
    intrinsics: CameraIntrinsics | None = None

    def __post_init__(self):
        if not 0 < self.d_min < self.d_max:
            raise ValueError(f"need 0 < d_min < d_max, got [{self.d_min}, {self.d_max}]")
        if not 1 <= self.levels <= 65535:
            raise ValueError(f"levels out of range: {self.levels}")
        self.codes = np.ascontiguousarray(self.codes, dtype=np.uint8 if self.levels <= 255 else np.uint16)
        if self.codes.ndim != 2:
            raise ValueError("codes must be 2-D")
        if self.codes.max(initial=0) > self.levels:
            raise ValueError(f"code {self.codes.max()} exceeds {self.levels} levels")

    @property
    def height(self) -> int:
        return self.codes.shape[0]

    @property
    def width(self) -> int:
        return self.codes.shape[1]


@dataclass(frozen=True)
class FieldPair:
    query_to_db: object
    db_to_query: object


@dataclass
class QueryJob:
    query_id: str
    intrinsics: CameraIntrinsics
    descriptor: np.ndarray
    fields: dict = field(default_factory=dict)
    k_loc: int = 10


# ----------------------------------------------------------------------------- device helpers
class _DeviceDepth:
    """One entry's stored depth resident in HBM + its vl_lift_depth record."""

    def __init__(self, depth, intr_db: CameraIntrinsics | None):
        import torch
        self.keep = []
        if hasattr(depth, "codes"):  # QuantizedDepthMap: decode through the reference table
            q = depth
            span = math.log(q.d_max / q.d_min)
            denom = max(q.levels - 1, 1)
            c = np.arange(q.levels + 1, dtype=np.float64)
            lut = (q.d_min * np.exp((c - 1.0) / denom * span)).astype(np.float32)
            lut[0] = 0.0
            codes = np.ascontiguousarray(q.codes)
            self.kind = KIND_CODE8 if codes.dtype == np.uint8 else KIND_CODE16
            vals = torch.from_numpy(codes.view(np.int16) if codes.dtype == np.uint16 else codes).cuda()
            self.lut = torch.from_numpy(lut).cuda()
            self.values, self.valid = vals, None
            h, w = codes.shape
            grid_intr = q.intrinsics
        else:
            v = np.asarray(depth.values)
            self.kind = KIND_F16 if v.dtype == np.float16 else KIND_F32
            v = np.ascontiguousarray(v, dtype=np.float16 if self.kind == KIND_F16 else np.float32)
            self.values = torch.from_numpy(v.view(np.int16) if self.kind == KIND_F16 else v).cuda()
            self.valid = torch.from_numpy(np.ascontiguousarray(depth.valid, dtype=np.uint8)).cuda()
            self.lut = None
            h, w = v.shape
            grid_intr = depth.intrinsics
        self.h, self.w = h, w
        self.grid_intr = grid_intr

    def record(self, intr_db, pose: Pose) -> _lib.LiftDepth:
        r = _lib.LiftDepth()
        r.width, r.height, r.kind = self.w, self.h, self.kind
        r.values = self.values.data_ptr()
        r.valid = self.valid.data_ptr() if self.valid is not None else None
        r.lut = self.lut.data_ptr() if self.lut is not None else None
        r.fx, r.fy, r.cx, r.cy = float(intr_db.fx), float(intr_db.fy), float(intr_db.cx), float(intr_db.cy)
        r.sx_depth = self.w / intr_db.width
        r.sy_depth = self.h / intr_db.height
        R = pose.R
        for i in range(9):
            r.R[i] = float(R.flat[i])
        for i in range(3):
            r.t[i] = float(pose.t[i])
        return r


def _check_span(fld, intr, what):
    if abs(fld.grid_w * fld.scale_x - intr.width) > 1e-6 * intr.width or \
       abs(fld.grid_h * fld.scale_y - intr.height) > 1e-6 * intr.height:
        raise ValueError(f"{what}: field grid {fld.grid_w}x{fld.grid_h} at scale "
                         f"({fld.scale_x}, {fld.scale_y}) does not span image {intr.width}x{intr.height}")


class _FieldUpload:
    """Device-side view of many fields for one vl_lift call.

    Planar fields (CorrespondenceField-like: targets/confidence arrays) are
    packed into two device arrays (one dtype per call: f64 if any planar
    field is f64).  IMLC fields (``FieldBlob``) are read in place from their
    arena's HBM mirror (one copy per arena, no repacking); their geometry
    comes from the arena's arrays, so big batches need no per-field work
    beyond one attribute read."""

    def __init__(self, fields, finish: bool = True):
        n = len(fields)
        self.fields = fields
        blob = np.fromiter((type(f) is FieldBlob for f in fields), dtype=bool, count=n)
        self.planar_idx = np.nonzero(~blob)[0]
        planar = [fields[i] for i in self.planar_idx]
        self.f64 = any(np.asarray(f.confidence).dtype != np.float32 or np.asarray(f.targets).dtype != np.float32
                       for f in planar)
        self.item = 8 if self.f64 else 4
        self.layout = np.where(blob, _lib.LIFT_IMLC, _lib.LIFT_PLANAR).astype(np.int32)
        self.tptr = np.zeros(n, dtype=np.uint64)
        self.cptr = np.zeros(n, dtype=np.uint64)
        self.gw = np.zeros(n, dtype=np.int64)
        self.gh = np.zeros(n, dtype=np.int64)
        self.sx = np.zeros(n, dtype=np.float64)
        self.sy = np.zeros(n, dtype=np.float64)
        self.keep = []
        self.bytes = 0
        self.groups = []  # (arena, field positions, record offsets inside the arena)
        blob_idx = np.nonzero(blob)[0]
        if blob_idx.size:
            arenas = {}
            for i in blob_idx:
                f = fields[i]
                arenas.setdefault(id(f.arena), (f.arena, []))[1].append(i)
            for arena, pos in arenas.values():
                pos = np.asarray(pos)
                fidx = np.fromiter((fields[i].index for i in pos), dtype=np.int64, count=pos.size)
                self.gw[pos], self.gh[pos] = arena.gw[fidx], arena.gh[fidx]
                self.sx[pos], self.sy[pos] = arena.sx[fidx], arena.sy[fidx]
                self.bytes += int(12 * (arena.gw[fidx] * arena.gh[fidx]).sum())
                self.groups.append((arena, pos, arena.roff[fidx]))
        if planar:
            self.gw[self.planar_idx] = [f.grid_w for f in planar]
            self.gh[self.planar_idx] = [f.grid_h for f in planar]
            self.sx[self.planar_idx] = [float(f.scale_x) for f in planar]
            self.sy[self.planar_idx] = [float(f.scale_y) for f in planar]
        self.targets = self.conf = None
        if finish:
            self.finish()

    def finish(self):
        """Device side: arena mirrors (waiting on side-stream uploads) and the
        planar fields' upload.  Host-only construction (``finish=False``) can
        run on a worker thread; this part runs on the launching thread."""
        import torch
        for arena, pos, roff in self.groups:
            dev = arena.device()
            arena.wait()  # a side-stream upload must land before the lift reads it
            self.keep.append(dev)
            self.tptr[pos] = np.uint64(dev.data_ptr()) + roff
        if self.planar_idx.size:
            dt = np.float64 if self.f64 else np.float32
            planar = [self.fields[i] for i in self.planar_idx]
            tg = [np.ascontiguousarray(f.targets, dtype=dt).reshape(-1) for f in planar]
            cf = [np.ascontiguousarray(f.confidence, dtype=dt).reshape(-1) for f in planar]
            t_off = np.concatenate([[0], np.cumsum([a.size for a in tg])]).astype(np.uint64)
            c_off = np.concatenate([[0], np.cumsum([a.size for a in cf])]).astype(np.uint64)
            self.targets = torch.from_numpy(np.concatenate(tg)).cuda()
            self.conf = torch.from_numpy(np.concatenate(cf)).cuda()
            self.tptr[self.planar_idx] = self.targets.data_ptr() + t_off[:-1] * self.item
            self.cptr[self.planar_idx] = self.conf.data_ptr() + c_off[:-1] * self.item
            self.bytes += int(self.targets.numel() + self.conf.numel()) * self.item
        return self

    @property
    def cells(self) -> int:
        return int((self.gw * self.gh).sum())


def _seg_table(q, e, d, dep, up: _FieldUpload) -> np.ndarray:
    """vl_lift_segment array (numpy structured) from per-segment arrays."""
    n = len(q)
    t = np.zeros(max(n, 1), dtype=_lib.LIFT_SEGMENT_DTYPE)
    if n:
        t["query"][:n], t["entry"][:n], t["direction"][:n], t["depth"][:n] = q, e, d, dep
        t["grid_w"][:n], t["grid_h"][:n] = up.gw, up.gh
        t["scale_x"][:n], t["scale_y"][:n] = up.sx, up.sy
        t["layout"][:n] = up.layout
        t["targets"][:n] = up.tptr
        t["confidence"][:n] = up.cptr
    return t


def _call_lift(table, nseg, deps, ndep, f64, threshold, mode, px, X, w, ent, cap, offs, flags, fields, ctx=None):
    ctx = ctx or _lib.context()
    rc = _lib.lib().vl_lift(ctx.handle, table.ctypes.data, nseg, deps, ndep, 1 if f64 else 0, float(threshold),
                            mode, px.data_ptr(), X.data_ptr(), w.data_ptr(), ent.data_ptr() if ent is not None else None,
                            cap,
                            offs.ctypes.data_as(C.POINTER(C.c_int64)), flags.ctypes.data_as(C.POINTER(C.c_int32)),
                            _lib.stream_ptr())
    ctx.check(rc, "vl_lift")
    bad = np.nonzero(flags[:nseg])[0]
    if bad.size:  # IMLC record content rules, checked on the GPU by the counting pass
        raise fields[int(bad[0])].content_error(int(flags[bad[0]]))


def _run_lift(segs_spec, depth_records, threshold, mode=0):
    """segs_spec: list of (query, entry, direction, depth_index, field).  Returns
    (px, X, w, None) CUDA tensors and host segment offsets."""
    import torch
    if not 0 <= threshold <= 1:
        raise ValueError(f"threshold must be in [0, 1], got {threshold}")
    _lib.context()
    n = len(segs_spec)
    fields = [s[4] for s in segs_spec]
    up = _FieldUpload(fields)
    table = _seg_table(*([x[k] for x in segs_spec] for k in range(4)), up)
    cap = max(up.cells, 1)
    deps = (_lib.LiftDepth * max(len(depth_records), 1))(*depth_records)
    px = torch.empty((cap, 2), dtype=torch.float64, device="cuda")
    X = torch.empty((cap, 3), dtype=torch.float64, device="cuda")
    w = torch.empty((cap,), dtype=torch.float64, device="cuda")
    offs = np.zeros(n + 1, dtype=np.int64)
    flags = np.zeros(max(n, 1), dtype=np.int32)
    # no per-match entry ids: every caller knows the entry of a segment (the
    # estimator never reads them), so the lift skips those 4 B per match
    _call_lift(table, n, deps, len(depth_records), up.f64, threshold, mode, px, X, w, None, cap, offs, flags,
               fields)
    tot = int(offs[-1])
    return px[:tot], X[:tot], w[:tot], None, offs, up


# ----------------------------------------------------------------------------- API
def dequantize_depth(q) -> DepthMap:
    """Codes -> f32 depth + validity on the GPU (mapstore.py:122-134)."""
    import torch
    dd = _DeviceDepth(q, None)
    ctx = _lib.context()
    vals = torch.empty((dd.h, dd.w), dtype=torch.float32, device="cuda")
    ok = torch.empty((dd.h, dd.w), dtype=torch.uint8, device="cuda")
    intr = q.intrinsics if q.intrinsics is not None else CameraIntrinsics(1.0, 1.0, 0.0, 0.0, q.width, q.height)
    rec = dd.record(intr, Pose.identity())
    rc = _lib.lib().vl_decode_depth(ctx.handle, C.byref(rec), vals.data_ptr(), ok.data_ptr(), _lib.stream_ptr())
    ctx.check(rc, "vl_decode_depth")
    return DepthMap(values=vals.cpu().numpy(), valid=ok.cpu().numpy().astype(bool), intrinsics=intr)


def interp_depth_many(depth, subpixels):
    """Bilinear depth at depth-map subpixels with the all-4-valid rule (localizer.py:87-115)."""
    import torch
    from .posest import _to_device
    pts = np.ascontiguousarray(np.asarray(subpixels, dtype=np.float64).reshape(-1, 2))
    n = pts.shape[0]
    dd = _DeviceDepth(depth, None)
    if dd.w < 2 or dd.h < 2:
        raise ValueError("depth map must be at least 2x2")
    ctx = _lib.context()
    dp = _to_device(pts)
    vals = torch.empty((max(n, 1),), dtype=torch.float64, device="cuda")
    ok = torch.empty((max(n, 1),), dtype=torch.uint8, device="cuda")
    rec = dd.record(CameraIntrinsics(1.0, 1.0, 0.0, 0.0, dd.w, dd.h), Pose.identity())
    rc = _lib.lib().vl_interp_depth(ctx.handle, C.byref(rec), dp.data_ptr(), n, vals.data_ptr(), ok.data_ptr(),
                                    _lib.stream_ptr())
    ctx.check(rc, "vl_interp_depth")
    return vals[:n].cpu().numpy(), ok[:n].cpu().numpy().astype(bool)


def interp_depth(depth, subpixel):
    v, ok = interp_depth_many(depth, np.asarray(subpixel, dtype=np.float64)[None])
    return float(v[0]) if ok[0] else None


def _entry_segments(query_job, entry, q_index, e_index, d_index):
    pair = query_job.fields[entry.id]
    intr_db = entry.intrinsics
    _check_span(pair.db_to_query, intr_db, f"entry {entry.id} db->query")
    _check_span(pair.query_to_db, query_job.intrinsics, f"entry {entry.id} query->db")
    return [(q_index, e_index, 0, d_index, pair.db_to_query), (q_index, e_index, 1, d_index, pair.query_to_db)]


def _device_depth(entry, depth, cache):
    """Device copy of an entry's stored depth, cached in `cache` (dict) by entry id;
    the caller keeps the cache alive until the lift has been enqueued."""
    key = getattr(entry, "id", None)
    dd = cache.get(key)
    if dd is None:
        dd = _DeviceDepth(depth, entry.intrinsics)
        cache[key] = dd
    return dd


def _depth_mismatch(entry, dd):
    """localizer.py:151-155 message when the depth map's image size differs from the entry's."""
    gi = dd.grid_intr
    if gi is not None and (gi.width != entry.intrinsics.width or gi.height != entry.intrinsics.height):
        return (f"entry {entry.id}: depth map covers {gi.width}x{gi.height}, "
                f"entry image is {entry.intrinsics.width}x{entry.intrinsics.height}")
    return None


def _depth_record(entry, depth, cache):
    """vl_lift_depth record of an entry (device copy cached in `cache`)."""
    dd = _device_depth(entry, depth, cache)
    msg = _depth_mismatch(entry, dd)
    if msg:
        raise ValueError(msg)
    return dd.record(entry.intrinsics, entry.pose)


def lift_arrays(query_job, entry, depth, threshold: float = CONFIDENCE_THRESHOLD):
    """Device (px, X, w) of one entry's lift (localizer.py:134-197 order)."""
    keep = {}
    segs = _entry_segments(query_job, entry, 0, 0, 0)  # span checks first (localizer.py:147-150)
    rec = _depth_record(entry, depth, keep)
    px, X, w, _, _, _ = _run_lift(segs, [rec], threshold)
    return px, X, w


def lift(query_job, entry, depth, threshold: float = CONFIDENCE_THRESHOLD) -> list:
    """Drop-in ``visloc.localizer.lift``: list of Match2D3D in reference order."""
    px, X, w = lift_arrays(query_job, entry, depth, threshold)
    P, Xh, wh = px.cpu().numpy(), X.cpu().numpy(), w.cpu().numpy()
    return [Match2D3D(P[i], Xh[i], float(wh[i]), entry.id) for i in range(wh.shape[0])]


def _failure(n):
    return PoseEstimate(pose=Pose.identity(), inlier_count=0, inlier_flags=np.zeros(n, dtype=bool),
                        score=math.inf, iterations=0, converged=False)


def _retrieve(jobs, index, retrieval):
    """Retrieved entry ids of every job: host (reference-exact numpy) or one GPU launch."""
    if index.size == 0:
        return [[] for _ in jobs]
    if retrieval == "host":
        return [[eid for eid, _ in index.topk(np.asarray(j.descriptor, dtype=np.float64), j.k_loc)] for j in jobs]
    if retrieval != "gpu":
        raise ValueError(f"retrieval must be 'host' or 'gpu', got {retrieval!r}")
    for j in jobs:
        if j.k_loc < 1:
            raise ValueError(f"k must be >= 1, got {j.k_loc}")
    kmax = max(j.k_loc for j in jobs)
    desc = np.stack([np.asarray(j.descriptor, dtype=np.float64).reshape(-1) for j in jobs])
    ids, _ = index.topk_batch(desc, kmax)
    return [row[: j.k_loc] for row, j in zip(ids, jobs)]


def _pair_fields(jobs, ranked_ids, by_id):
    """Host half of the plan (no device work; safe on a worker thread): every
    (query, retrieved entry) pair with fields, in the reference's order
    (sorted retrieved ids, localizer.py:220-235), and the fields' geometry."""
    pq, peid, fields, spans = [], [], [], []
    for qi, (job, ranked) in enumerate(zip(jobs, ranked_ids)):
        qI = job.intrinsics
        for eid in sorted(ranked):
            pair = job.fields.get(eid)
            if pair is None:
                continue
            eI = by_id[eid].intrinsics
            pq.append(qi)
            peid.append(eid)
            fields += (pair.db_to_query, pair.query_to_db)
            spans += ((eI.width, eI.height), (qI.width, qI.height))
    return pq, peid, fields, spans, _FieldUpload(fields, finish=False)


def _plan_finish(pairs, by_id, depth_cache, device_cache):
    """Device half: depth records (decoded depth cached in HBM), arena
    waits, and the reference's per-entry checks in its order (db->query
    span, query->db span, depth size; localizer.py:147-155)."""
    pq, peid, fields, spans, up = pairs
    recs, rec_of, err_of, pe, derr = [], {}, {}, [], []
    for eid in peid:
        k = rec_of.get(eid)
        if k is None:
            entry = by_id[eid]
            if depth_cache is not None and eid in depth_cache:
                depth = depth_cache[eid]
            else:
                if getattr(entry, "qdepth", None) is None:
                    raise ValueError(f"entry {eid} has no stored depth")
                depth = entry.qdepth
            dd = _device_depth(entry, depth, device_cache)
            k = rec_of[eid] = len(recs)
            recs.append(dd.record(entry.intrinsics, entry.pose))
            err_of[eid] = _depth_mismatch(entry, dd)
        pe.append(k)
        derr.append(err_of[eid])
    n = len(pq)
    if n:
        WH = np.array(spans, dtype=np.float64).reshape(-1, 2)
        bad = (np.abs(up.gw * up.sx - WH[:, 0]) > 1e-6 * WH[:, 0]) | \
              (np.abs(up.gh * up.sy - WH[:, 1]) > 1e-6 * WH[:, 1])
        bad_pair = bad.reshape(-1, 2).any(axis=1) | np.fromiter((m is not None for m in derr), bool, n)
        if bad_pair.any():
            k = int(np.argmax(bad_pair))
            for j, what in ((2 * k, "db->query"), (2 * k + 1, "query->db")):
                if bad[j]:
                    f, (w, h) = fields[j], spans[j]
                    raise ValueError(f"entry {peid[k]} {what}: field grid {f.grid_w}x{f.grid_h} at scale "
                                     f"({f.scale_x}, {f.scale_y}) does not span image {w}x{h}")
            raise ValueError(derr[k])
    up.finish()
    q = np.repeat(np.asarray(pq, dtype=np.int64), 2)
    e = np.repeat(np.asarray(pe, dtype=np.int64), 2)
    d = np.tile(np.array([0, 1], dtype=np.int64), n)
    return q, e, d, fields, up, recs


def _index_of(vmap, index):
    if index is None:
        index = DescriptorIndex.from_entries((e.id, e.descriptor) for e in vmap.entries)
    return index


def _plan(jobs, vmap, index, depth_cache, device_cache, retrieval="host", ranked=None):
    """Segment arrays + depth records for every query."""
    by_id = {e.id: e for e in vmap.entries}
    if ranked is None:
        ranked = _retrieve(jobs, _index_of(vmap, index), retrieval)
    return _plan_finish(_pair_fields(jobs, ranked, by_id), by_id, depth_cache, device_cache)


class LiftPlan:
    """A query set's fields and depth resident in HBM, ready to lift + estimate.

    Construction does the host work once (retrieval ranking, field/depth
    upload, segment table); ``lift()`` / ``run_device()`` then run entirely
    on the GPU and can be repeated (the device-resident throughput path).
    """

    def __init__(self, jobs, vmap, index=None, depth_cache=None, device_cache=None,
                 threshold: float = CONFIDENCE_THRESHOLD, retrieval: str = "host", pairs=None, ctx=None):
        import torch
        self.ctx = ctx  # explicit _lib.Context (own workspace) for concurrent lanes
        if not 0 <= threshold <= 1:
            raise ValueError(f"threshold must be in [0, 1], got {threshold}")
        self.jobs = list(jobs)
        self.threshold = float(threshold)
        self.device_cache = {} if device_cache is None else device_cache
        if pairs is None:  # ``pairs``: a precomputed ``_pair_fields`` (the pipelined loop's worker)
            q, e, d, self.fields, self.up, recs = _plan(self.jobs, vmap, index, depth_cache, self.device_cache,
                                                         retrieval)
        else:
            q, e, d, self.fields, self.up, recs = _plan_finish(pairs, {x.id: x for x in vmap.entries},
                                                                depth_cache, self.device_cache)
        self.nseg = len(self.fields)
        self.seg_q = q
        self.table = _seg_table(q, e, d, e, self.up)
        cap = self.up.cells
        self.ndep = len(recs)
        self.deps = (_lib.LiftDepth * max(self.ndep, 1))(*recs)
        self.cap = max(cap, 1)
        self.px = torch.empty((self.cap, 2), dtype=torch.float64, device="cuda")
        self.X = torch.empty((self.cap, 3), dtype=torch.float64, device="cuda")
        self.w = torch.empty((self.cap,), dtype=torch.float64, device="cuda")
        self.offs = np.zeros(self.nseg + 1, dtype=np.int64)
        self.flags = np.zeros(max(self.nseg, 1), dtype=np.int32)
        self.cells = cap
        self.field_bytes = self.up.bytes

    def lift(self):
        """Run the lift; returns per-query [start, end) match ranges (host)."""
        with _lib.nvtx(f"visloc.lift segments={self.nseg}"):
            _call_lift(self.table, self.nseg, self.deps, self.ndep, self.up.f64, self.threshold, 0, self.px, self.X,
                       self.w, None, self.cap, self.offs, self.flags, self.fields, self.ctx)
        qs = np.arange(len(self.jobs))
        # segments are in query order: first/last segment of every query
        start = self.offs[np.searchsorted(self.seg_q, qs, "left")]
        end = self.offs[np.searchsorted(self.seg_q, qs, "right")]
        return start, end

    def run_device(self, cfg: RansacConfig, seeds=None, out=None, ranges=None):
        """Lift (unless ``ranges`` from an earlier ``lift()`` are given) + batched
        estimator, all on device.  Returns (out dict or None, estimated query
        indices, their match offsets, per-query ranges)."""
        import torch
        Q = len(self.jobs)
        seeds = [cfg.seed] * Q if seeds is None else list(seeds)
        start, end = self.lift() if ranges is None else ranges
        run = [qi for qi in range(Q) if end[qi] - start[qi] >= 3]
        if not run:
            return None, run, None, (start, end)
        offsets = np.concatenate([[0], np.cumsum([end[qi] - start[qi] for qi in run])]).astype(np.int64)
        if all(start[run[i + 1]] == end[run[i]] for i in range(len(run) - 1)):
            a, b = int(start[run[0]]), int(end[run[-1]])
            dpx, dX, dw = self.px[a:b], self.X[a:b], self.w[a:b]
        else:
            sl = [slice(int(start[qi]), int(end[qi])) for qi in run]
            dpx = torch.cat([self.px[s] for s in sl]).contiguous()
            dX = torch.cat([self.X[s] for s in sl]).contiguous()
            dw = torch.cat([self.w[s] for s in sl]).contiguous()
        res = ransac_pnp_device(dpx, dX, dw, offsets, [self.jobs[qi].intrinsics for qi in run],
                                [seeds[qi] for qi in run], cfg, out=out, ctx=self.ctx)
        return res, run, offsets, (start, end)

    def localize(self, cfg: RansacConfig, seeds=None) -> list:
        return self.collect(*self.run_device(cfg, seeds))

    def collect(self, out, run, offsets, ranges, host=None) -> list:
        """PoseEstimates of a ``run_device`` result (``host``: its arrays
        already copied out by ``_stage_results``)."""
        start, end = ranges
        res: list = [None] * len(self.jobs)
        for qi in range(len(self.jobs)):
            if qi not in run:
                res[qi] = _failure(int(end[qi] - start[qi]))
        if run:
            ests = _estimates_from(out, offsets) if host is None else _estimates_from_host(*host)
            for qi, est in zip(run, ests):
                res[qi] = est
        return res


def localize_batch(jobs, vmap, cfg: RansacConfig, seeds=None, index=None, depth_cache=None,
                   confidence_threshold: float = CONFIDENCE_THRESHOLD, device_cache=None,
                   retrieval: str = "host"):
    """Retrieve, lift (one GPU launch sequence for every query) and estimate every pose.

    Each query behaves like ``localize(job, vmap, RansacConfig(seed=seeds[i]))``.
    ``device_cache`` (dict) keeps decoded depth resident in HBM across calls.
    ``retrieval="gpu"`` ranks all queries in one ``vl_retrieval_topk`` launch
    (ids equal the host ranking except on near-exact similarity ties).
    """
    jobs = list(jobs)
    if not jobs:
        return []
    plan = LiftPlan(jobs, vmap, index, depth_cache, device_cache, confidence_threshold, retrieval)
    return plan.localize(cfg, seeds)


_LANE_CONTEXTS: dict = {}


def serving_schedule(Q: int):
    """Micro-batch ends for ``localize_pipelined`` when the fields' PCIe copy
    dominates (C5: 0.84 GB of IMLC records per 256 queries, ~15 ms at
    55 GB/s against ~10 ms of GPU work): a small first batch so the GPU
    starts early, a small last batch so little work trails the last copy,
    larger batches between (weights 1,3,4,4,3,1 / 16; tools/c5_host_breakdown.py
    sweep).  Small query counts collapse to fewer batches."""
    w = np.array([1, 3, 4, 4, 3, 1], dtype=np.float64)
    ends = np.round(np.cumsum(w) / w.sum() * Q).astype(np.int64)
    return sorted({int(e) for e in ends if e > 0} | {Q})


def _lanes(device: int, n: int):
    """``n`` (library context, stream) lanes of a device and a copy stream,
    kept for reuse: fresh streams would start with empty allocator pools."""
    import torch
    lst = _LANE_CONTEXTS.setdefault(device, [])
    with torch.cuda.device(device):
        while len(lst) < n:
            lst.append((_lib.Context(device), torch.cuda.Stream()))
        copy = _LANE_CONTEXTS.get(("copy", device))
        if copy is None:
            copy = _LANE_CONTEXTS[("copy", device)] = torch.cuda.Stream()
    return lst[:n], copy


def localize_pipelined(batches, vmap, cfg: RansacConfig, seeds=None, index=None, depth_cache=None,
                       confidence_threshold: float = CONFIDENCE_THRESHOLD, device_cache=None,
                       retrieval: str = "host", buffers=None, lanes: int | None = None):
    """Micro-batched serving loop: ``batches`` = [(jobs, arena), ...], each
    batch's IMLC fields in its own ``FieldArena``.

    Every query is retrieved up front (one ranking call) and the map depth
    it needs is made resident; then ``lanes`` host threads (default 2, env
    VISLOC_PIPE_LANES), each with its own stream and library context, take
    batches round-robin: plan, lift, estimate, read back.  While one lane
    sits in the library's round loop (GIL released) the other plans its
    next batch and the GPU runs both lanes' kernels concurrently.  Batch k's
    fields go to HBM on a copy stream into ``buffers[k % len(buffers)]``
    once batch k - len(buffers) has been lifted.  Each query behaves like
    ``localize(job, vmap, RansacConfig(seed=seeds[i]))``.
    ``buffers`` (optional): uint8 CUDA tensors large enough for any arena,
    reused across calls (default: one per lane + 1).  ``seeds`` covers all
    jobs, in order.  Returns the flat list of PoseEstimates."""
    import threading

    import torch
    batches = list(batches)
    if not batches:
        return []
    if not 0 <= confidence_threshold <= 1:
        raise ValueError(f"threshold must be in [0, 1], got {confidence_threshold}")
    nb = len(batches)
    L = max(1, min(int(lanes or os.environ.get("VISLOC_PIPE_LANES", 2)), nb))
    njobs = sum(len(j) for j, _ in batches)
    seeds = [cfg.seed] * njobs if seeds is None else list(seeds)
    if buffers is None:
        big = max(a.host.numel() for _, a in batches)
        buffers = [torch.empty(big, dtype=torch.uint8, device="cuda") for _ in range(min(L + 1, nb))]
    B = len(buffers)
    all_jobs = [j for jobs, _ in batches for j in jobs]
    first = np.cumsum([0] + [len(j) for j, _ in batches])
    dev = torch.cuda.current_device()
    lanes_, copy = _lanes(dev, L)
    ctxs, streams = [c for c, _ in lanes_], [st for _, st in lanes_]
    comp = torch.cuda.current_stream()
    copy.wait_stream(comp)
    lifted = [torch.cuda.Event() for _ in batches]
    issued = [threading.Event() for _ in batches]
    results, errors = [None] * nb, [None] * nb
    lock = threading.Lock()

    def upload(k):
        if k < nb:
            with lock:
                if k >= B:
                    copy.wait_event(lifted[k - B])  # buffer k % B was last read by batch k - B
                batches[k][1].upload(buffers[k % B], stream=copy)
            issued[k].set()

    for k in range(min(B, nb)):  # the first payloads cross PCIe while the queries are ranked
        upload(k)
    ranked = _retrieve(all_jobs, _index_of(vmap, index), retrieval)
    by_id = {e.id: e for e in vmap.entries}
    device_cache = {} if device_cache is None else device_cache
    for job, ids in zip(all_jobs, ranked):  # depth the lanes will read, resident before they start
        for eid in ids:
            if eid in job.fields and eid not in device_cache:
                entry = by_id[eid]
                depth = depth_cache.get(eid) if depth_cache is not None else None
                depth = depth if depth is not None else getattr(entry, "qdepth", None)
                if depth is not None:
                    _device_depth(entry, depth, device_cache)
    for st in streams:
        st.wait_stream(comp)

    order = iter(range(nb))  # a free lane takes the next batch

    def lane(i):
        with torch.cuda.device(dev), torch.cuda.stream(streams[i]):
            while True:
                with lock:
                    k = next(order, None)
                if k is None:
                    return
                issued[k].wait()
                if any(e is not None for e in errors):
                    continue
                try:
                    jobs = batches[k][0]
                    pk = _pair_fields(jobs, ranked[first[k]:first[k + 1]], by_id)
                    plan = LiftPlan(jobs, vmap, None, depth_cache, device_cache, confidence_threshold, pairs=pk,
                                    ctx=ctxs[i])
                    ranges = plan.lift()
                    lifted[k].record(streams[i])
                    upload(k + B)
                    out, run, offsets, ranges = plan.run_device(cfg, seeds[first[k]:first[k + 1]], ranges=ranges)
                    host = _stage_results(out, offsets) if run else None
                    results[k] = plan.collect(out, run, offsets, ranges, host)
                except BaseException as exc:  # noqa: BLE001 - re-raised on the calling thread
                    errors[k] = exc
                    for j in range(k + 1, nb):  # release every lane still waiting on an upload
                        issued[j].set()

    if L == 1:
        lane(0)
    else:
        threads = [threading.Thread(target=lane, args=(i,), daemon=True) for i in range(L)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    for st in streams:
        comp.wait_stream(st)
    comp.wait_stream(copy)
    for exc in errors:
        if exc is not None:
            raise exc
    return [est for r in results for est in r]


def localize(query_job, vmap, cfg: RansacConfig, index=None, depth_cache=None,
             confidence_threshold: float = CONFIDENCE_THRESHOLD) -> PoseEstimate:
    """Drop-in ``visloc.localizer.localize`` (localizer.py:200-238)."""
    return localize_batch([query_job], vmap, cfg, seeds=[cfg.seed], index=index, depth_cache=depth_cache,
                          confidence_threshold=confidence_threshold)[0]
