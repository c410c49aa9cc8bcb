"""Confidence-weighted LO-RANSAC PnP — drop-in for ``visloc.posest``.

Same public surface as ``pkg/src/visloc/posest.py``: ``Match2D3D`` (:55-66),
``RansacConfig`` (:69-90), ``PoseEstimate`` (:93-103),
``UnderConstrainedError`` (:51-52), ``required_iterations`` (:106-120),
``msac_score`` (:160-175) and ``ransac_pnp`` (:223-299), plus the additive
``ransac_pnp_batch`` / ``ransac_pnp_device`` for many queries per launch.

Every estimator call runs on the GPU through the sm_100a C ABI
(``vl_ransac_pnp`` / ``vl_msac_score``); the host only packs arrays, moves
them to HBM and unpacks results.  Identical inputs and config (seed
included) reproduce the reference's minimal sample sets exactly.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import os
import time

from . import _lib
from .geometry import CameraIntrinsics, Pose

__all__ = [
    "Match2D3D", "PoseEstimate", "RansacConfig", "UnderConstrainedError", "msac_score",
    "ransac_pnp", "ransac_pnp_batch", "ransac_pnp_device", "ransac_pnp_host", "ransac_pnp_stream",
    "required_iterations",
]


class UnderConstrainedError(ValueError):
    """Fewer correspondences than the minimal sample size."""


@dataclass(frozen=True)
class Match2D3D:
    query_px: np.ndarray
    world_point: np.ndarray
    weight: float
    entry_id: str = ""

    def __post_init__(self):
        if not self.weight > 0:
            raise ValueError(f"match weight must be positive, got {self.weight}")


@dataclass(frozen=True)
class RansacConfig:
    max_iterations: int = 100_000
    batch_size: int = 1_000
    miss_probability: float = 1e-4
    reproj_threshold: float = 12.0
    max_scoring: int = 10_000
    cauchy_scale: float | None = None
    lm_max_iters: int = 100
    seed: int = 0

    def __post_init__(self):
        if self.reproj_threshold <= 0:
            raise ValueError("reproj_threshold must be positive")
        if not 0 < self.miss_probability < 1:
            raise ValueError("miss_probability must be in (0, 1)")
        if self.batch_size > self.max_iterations:
            raise ValueError("batch_size must not exceed max_iterations")

    @property
    def cauchy(self) -> float:
        return self.reproj_threshold if self.cauchy_scale is None else self.cauchy_scale


@dataclass
class PoseEstimate:
    pose: Pose
    inlier_count: int
    inlier_flags: np.ndarray
    score: float
    iterations: int
    converged: bool
    stats: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        self.inlier_flags = np.asarray(self.inlier_flags, dtype=bool)


def required_iterations(inlier_ratio: float, miss_probability: float, sample_size: int = 3,
                        max_iterations: int = 100_000) -> int:
    """Adaptive bound ceil(ln eta / ln(1 - eps^m)), clamped (posest.py:106-120)."""
    eps = min(max(inlier_ratio, 0.0), 1.0)
    if eps <= 0.0:
        return max_iterations
    if eps >= 1.0:
        return 1
    den = math.log1p(-(eps ** sample_size))
    if den == 0.0:
        return max_iterations
    return int(min(max(math.ceil(math.log(miss_probability) / den), 1), max_iterations))


# ----------------------------------------------------------------- helpers
def _host_arrays(matches):
    """Match list or (px, X, w) triple -> fp64 numpy (n,2), (n,3), (n,) (posest.py:123-134)."""
    if isinstance(matches, tuple) and len(matches) == 3:
        px, X, w = matches
        if hasattr(px, "detach"):  # torch tensors
            px, X, w = (a.detach().cpu().numpy() for a in (px, X, w))
        return (np.ascontiguousarray(np.asarray(px, dtype=np.float64).reshape(-1, 2)),
                np.ascontiguousarray(np.asarray(X, dtype=np.float64).reshape(-1, 3)),
                np.ascontiguousarray(np.asarray(w, dtype=np.float64).reshape(-1)))
    px = np.array([m.query_px for m in matches], dtype=np.float64).reshape(-1, 2)
    X = np.array([m.world_point for m in matches], dtype=np.float64).reshape(-1, 3)
    w = np.array([m.weight for m in matches], dtype=np.float64).reshape(-1)
    return px, X, w


def _intr_c(intr) -> _lib.Intrinsics:
    return _lib.Intrinsics(float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy))


def _cfg_c(cfg: RansacConfig) -> _lib.RansacConfigC:
    c = _lib.RansacConfigC()
    c.max_iterations = int(cfg.max_iterations)
    c.batch_size = int(cfg.batch_size)
    c.max_scoring = int(cfg.max_scoring)
    c.miss_probability = float(cfg.miss_probability)
    c.reproj_threshold = float(cfg.reproj_threshold)
    c.cauchy_scale = float(cfg.cauchy) if cfg.cauchy_scale is not None else -1.0
    c.lm_max_iters = int(cfg.lm_max_iters)
    return c


def _to_device(a: np.ndarray):
    import torch
    _lib.context()  # fails loudly (VislocError) without a CUDA device / built library
    t = torch.from_numpy(np.ascontiguousarray(a))
    if t.numel() == 0:
        return t.cuda()
    return t.pin_memory().cuda(non_blocking=True)


# ----------------------------------------------------------------- device entry
def ransac_pnp_device(px, X, w, offsets, intrinsics, seeds, cfg: RansacConfig, out=None, stages=None, ctx=None):
    """Batched estimator on device-resident inputs (the HBM-resident hot path).

    ``px`` (N,2), ``X`` (N,3), ``w`` (N,) are fp64 CUDA tensors holding Q
    queries back to back; ``offsets`` (Q+1,) int64 host array; ``intrinsics``
    a list of Q intrinsics; ``seeds`` Q seeds (each query behaves exactly like
    ``ransac_pnp`` with ``RansacConfig(seed=seeds[i])``).  Returns a dict of
    CUDA tensors (q, t, flags, count, score, iterations, converged, stats).
    ``stages``: optional ``(stage_end, events)`` — the inputs of queries
    ``[stage_end[k-1], stage_end[k])`` are only valid once ``events[k]``
    (``torch.cuda.Event``) completes (``vl_ransac_pnp_staged``).  ``ctx``: an
    explicit ``_lib.Context`` (default: the device's shared one).
    """
    import torch
    offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    Q = offsets.shape[0] - 1
    if Q <= 0:
        raise ValueError("need at least one query")
    counts = np.diff(offsets)
    if counts.min() < 3:
        raise UnderConstrainedError(f"need >= 3 matches, got {int(counts[np.argmax(counts < 3)])}")
    dev = px.device
    N = int(offsets[-1])
    for a, shape in ((px, (N, 2)), (X, (N, 3)), (w, (N,))):
        if not (a.is_cuda and a.dtype == torch.float64 and a.is_contiguous() and tuple(a.shape) == shape):
            raise ValueError(f"expected contiguous fp64 CUDA tensor of shape {shape}")
    if ctx is None:  # an explicit context (own workspace) lets several runs proceed concurrently
        ctx = _lib.context(dev.index)
    if out is None:
        out = _result_block(Q, N, dev)
    intr_arr = (_lib.Intrinsics * Q)(*[_intr_c(i) for i in intrinsics])
    rng_arr = (_lib.PCG64State * Q)(*[_lib.pcg64_state(int(s)) for s in seeds])
    args = _lib.RansacArgs()
    args.num_queries = Q
    args.offsets = offsets.ctypes.data_as(C.POINTER(C.c_int64))
    args.intr = intr_arr
    args.rng = rng_arr
    args.px, args.X, args.w = px.data_ptr(), X.data_ptr(), w.data_ptr()
    args.cfg = _cfg_c(cfg)
    o = _lib.RansacOut()
    o.q, o.t, o.inlier_flags = out["q"].data_ptr(), out["t"].data_ptr(), out["flags"].data_ptr()
    o.inlier_count, o.score = out["count"].data_ptr(), out["score"].data_ptr()
    o.iterations, o.converged = out["iterations"].data_ptr(), out["converged"].data_ptr()
    o.stats = out["stats"].data_ptr()
    with torch.cuda.device(dev), _lib.nvtx(f"visloc.ransac_pnp_device Q={Q}"):
        if stages is None:
            rc = _lib.lib().vl_ransac_pnp(ctx.handle, C.byref(args), C.byref(o), _lib.stream_ptr())
        else:
            ends, events = stages
            ends_c = (C.c_int32 * len(ends))(*[int(e) for e in ends])
            evs_c = (C.c_void_p * len(events))(*[ev.cuda_event for ev in events])
            rc = _lib.lib().vl_ransac_pnp_staged(ctx.handle, C.byref(args), C.byref(o), len(ends), ends_c, evs_c,
                                                 _lib.stream_ptr())
    ctx.check(rc, "vl_ransac_pnp_staged" if stages is not None else "vl_ransac_pnp")
    return out


_RESULT_LAYOUT = (("q", "float64", 4), ("t", "float64", 3), ("score", "float64", 1), ("count", "int64", 1),
                  ("iterations", "int64", 1), ("stats", "int64", 4), ("converged", "int32", 1))


def _result_block(Q: int, N: int, dev):
    """The result dict of Q queries / N matches as views of ONE device
    allocation (8-B aligned fields, the flags last), so that a single
    device-to-host copy returns everything (_stage_results)."""
    import torch
    sizes = [(k, getattr(torch, dt), Q * m) for k, dt, m in _RESULT_LAYOUT]
    off, spans = 0, []
    for k, dt, n in sizes:
        spans.append((k, dt, off, n))
        off += (n * torch.empty((), dtype=dt).element_size() + 7) // 8 * 8
    block = torch.empty((off + N,), dtype=torch.uint8, device=dev)
    out = {}
    for k, dt, o, n in spans:
        v = block[o:o + n * torch.empty((), dtype=dt).element_size()].view(dt)
        out[k] = v.view(Q, -1) if k in ("q", "t", "stats") else v
    out["flags"] = block[off:off + N]
    return out


def _stage_results(out, offsets):
    """Enqueue the D2H copies of a device result dict into pinned host
    tensors on the current stream; returns (host dict, ready event, offsets).
    A dict from _result_block (every field in one allocation) takes ONE copy
    (the drop-in ransac_pnp: 8 -> 1 transfers per call)."""
    import torch
    keys = ("q", "t", "flags", "count", "score", "iterations", "converged", "stats")
    host = {}
    st = out["q"].untyped_storage()
    base = st.data_ptr()
    if all(out[k].untyped_storage().data_ptr() == base and out[k].is_contiguous() for k in keys):
        dev_all = torch.empty((0,), dtype=torch.uint8, device=out["q"].device).set_(st)
        h_all = torch.empty((st.nbytes(),), dtype=torch.uint8, pin_memory=True)
        h_all.copy_(dev_all, non_blocking=True)
        for k in keys:
            v = out[k]
            o = v.data_ptr() - base
            host[k] = h_all[o:o + v.numel() * v.element_size()].view(v.dtype).view(v.shape)
    else:
        for k in keys:
            v = out[k]
            h = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
            h.copy_(v, non_blocking=True)
            host[k] = h
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream())
    return host, ev, offsets


def _estimates_from_host(host, ev, offsets) -> list[PoseEstimate]:
    """PoseEstimates once ``_stage_results``' copies land (any thread): the
    flags are viewed as bool without a conversion pass and per-query masks
    are views of the one host flag array."""
    ev.synchronize()
    q, t = host["q"].numpy(), host["t"].numpy()
    flags = host["flags"].numpy().view(np.bool_)
    cnt, score = host["count"].numpy().tolist(), host["score"].numpy().tolist()
    iters, conv = host["iterations"].numpy().tolist(), host["converged"].numpy().tolist()
    stats = host["stats"].numpy().tolist()
    offs = np.asarray(offsets).tolist()
    res = []
    for i in range(q.shape[0]):
        st = stats[i]
        res.append(PoseEstimate(
            pose=Pose._trusted(q[i], t[i]), inlier_count=cnt[i], inlier_flags=flags[offs[i]:offs[i + 1]],
            score=score[i], iterations=iters[i], converged=bool(conv[i]),
            stats={"lo_calls": st[0], "hypotheses": st[1], "evals": st[2], "rounds": st[3]}))
    return res


def _estimates_from(out, offsets) -> list[PoseEstimate]:
    """PoseEstimates from the device result dict (one pinned D2H per array)."""
    return _estimates_from_host(*_stage_results(out, offsets))


def _host_chunks(Q: int, chunk_queries=None):
    """Query chunks of the host pipeline.

    Fixed ``chunk_queries`` gives equal chunks.  The default is a doubling
    schedule (Q/16, Q/8, Q/4, ... , rest): only the first, small chunk's copy
    is exposed, each chunk's estimation covers the next chunk's (twice as
    large) host-to-device copy, and the bulk of the queries still run in
    large, well-occupied batches.
    """
    if chunk_queries:
        return [(q0, min(Q, q0 + chunk_queries)) for q0 in range(0, Q, chunk_queries)]
    chunks, q0, size = [], 0, max(1, -(-Q // 16))
    while q0 < Q:
        q1 = Q if Q - q0 < 3 * size else q0 + size  # fold a short remainder into the last chunk
        chunks.append((q0, q1))
        q0, size = q1, 2 * size
    return chunks


def _stage_schedule(Q: int):
    """Staged-admission stage ends: Q/16, then doubling stage sizes (Q/8, Q/4, ...),
    a short remainder folded into the last stage.  Each admission adds one
    LO-heavy first round to the shared loop, so few stages beat many small
    ones (C3 sweep, tools/host_pipe.py: [63, 189, 441, 1000] is the best of the
    schedules tried)."""
    ends, q0, size = [], 0, max(1, -(-Q // 16))
    while q0 < Q:
        q1 = Q if Q - q0 < 3 * size // 2 else q0 + size
        ends.append(q1)
        q0, size = q1, 2 * size
    return ends


def ransac_pnp_host(px, X, w, offsets, intrinsics, seeds, cfg: RansacConfig, chunk_queries=None,
                    stage_ends=None):
    """Batched estimator on HOST buffers: H2D copy, device run, D2H of the results.

    ``px``/``X``/``w`` are packed host arrays (numpy, or pinned torch CPU
    tensors for full-bandwidth copies).  Default: the inputs are copied in
    stages (``_stage_schedule``) on a side stream and ONE estimator run
    admits each stage's queries as soon as its copy lands
    (``vl_ransac_pnp_staged``), so PCIe traffic overlaps estimation without
    splitting the run.  ``chunk_queries=k`` instead runs separate estimator
    calls on chunks of k queries, double-buffered (``_host_chunks``).
    Returns a dict of numpy arrays (q, t, flags, count, score, iterations,
    converged, stats) and the byte counts moved each way.
    """
    import torch
    _lib.context()
    offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    Q = offsets.shape[0] - 1
    N = int(offsets[-1])
    host_in = []
    for a in (px, X, w):
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        if not t.is_pinned():
            t = t.pin_memory()
        host_in.append(t)
    intrinsics = list(intrinsics)
    seeds = list(seeds)
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    dev = torch.device("cuda", torch.cuda.current_device())
    out = {
        "q": torch.empty((Q, 4), dtype=torch.float64, device=dev),
        "t": torch.empty((Q, 3), dtype=torch.float64, device=dev),
        "flags": torch.empty((max(N, 1),), dtype=torch.uint8, device=dev),
        "count": torch.empty((Q,), dtype=torch.int64, device=dev),
        "score": torch.empty((Q,), dtype=torch.float64, device=dev),
        "iterations": torch.empty((Q,), dtype=torch.int64, device=dev),
        "converged": torch.empty((Q,), dtype=torch.int32, device=dev),
        "stats": torch.empty((Q, 4), dtype=torch.int64, device=dev),
    }
    # pinned result buffers from the pool (a fresh pinned allocation costs up
    # to tens of ms; a set is reused once the caller has dropped its arrays)
    pset = _PINNED_POOL.get({k: (tuple(v.shape), v.dtype) for k, v in out.items()})
    host_out = pset.tensors
    if not chunk_queries:
        with _lib.nvtx(f"visloc.ransac_pnp_host Q={Q}"):
            ends = list(stage_ends) if stage_ends is not None else _stage_schedule(Q)
            bufs = [torch.empty(t.shape, dtype=t.dtype, device=dev) for t in host_in]
            events = []
            copy.wait_stream(comp)  # the device buffers are fresh allocations on the compute stream
            with torch.cuda.stream(copy):
                q0 = 0
                for q1 in ends:
                    r0, r1 = int(offsets[q0]), int(offsets[q1])
                    for dst, src in zip(bufs, host_in):
                        dst[r0:r1].copy_(src[r0:r1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy)
                    events.append(ev)
                    q0 = q1
            ransac_pnp_device(bufs[0], bufs[1], bufs[2], offsets, intrinsics, seeds, cfg, out=out,
                              stages=(ends, events))
            for key, v in out.items():
                host_out[key].copy_(v[:N] if key == "flags" else v, non_blocking=True)
            comp.synchronize()
    else:
        _host_pipeline_chunks(host_in, offsets, intrinsics, seeds, cfg, chunk_queries, out, host_out, comp, copy,
                              dev)
    full = {k: v.numpy() for k, v in host_out.items()}
    pset.hand_out(full.values())  # views below keep these alive while the caller holds them
    host = {k: v[:N] if k == "flags" else v for k, v in full.items()}
    h2d_bytes = sum(int(t.numel() * t.element_size()) for t in host_in)
    d2h_bytes = sum(int(v.nbytes) for v in host.values())
    return host, h2d_bytes, d2h_bytes


_STREAM_DEBUG = bool(os.environ.get("VISLOC_STREAM_DEBUG"))


def ransac_pnp_stream(batches, cfg: RansacConfig):
    """Serve a sequence of query batches held in HOST memory (generator; the serving loop).

    ``batches``: iterable of ``(px, X, w, offsets, intrinsics, seeds)`` — the
    arguments of ``ransac_pnp_host`` (pinned torch CPU tensors for full PCIe
    bandwidth).  Yields ``(results, h2d_bytes, d2h_bytes)`` per batch, in
    order, ``results`` as ``ransac_pnp_host`` returns them.

    Batch k+1's inputs are copied to HBM on a side stream while batch k is
    estimated (two device input buffers), so after the first batch — which is
    admitted stage by stage like ``ransac_pnp_host`` — a steady stream runs at
    the estimator's device-resident rate whenever the PCIe copy of a batch is
    shorter than its estimation.  Every batch's H2D and its results' D2H are
    real copies; nothing is cached between batches.
    """
    import torch
    _lib.context()
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    dev = torch.device("cuda", torch.cuda.current_device())
    bufs = [None, None]       # device input sets (px, X, w), alternating
    freed = [None, None]      # event: the run that read the set has finished
    copy.wait_stream(comp)

    def prepare(b):
        px, X, w, offsets, intrinsics, seeds = b
        offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
        host_in = []
        for a in (px, X, w):
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
            if not t.is_pinned():
                t = t.pin_memory()
            host_in.append(t)
        return host_in, offsets, list(intrinsics), list(seeds)

    def h2d(k, host_in, offsets, staged):
        """Enqueue batch k's copy into buffer set k % 2; returns (stage ends, events)."""
        j = k % 2
        if bufs[j] is None or any(bd.shape != hs.shape for bd, hs in zip(bufs[j], host_in)):
            with torch.cuda.stream(copy):
                if freed[j] is not None:
                    copy.wait_event(freed[j])
                bufs[j] = [torch.empty(t.shape, dtype=t.dtype, device=dev) for t in host_in]
        Q = offsets.shape[0] - 1
        ends = _stage_schedule(Q) if staged else [Q]
        events = []
        with torch.cuda.stream(copy):
            if freed[j] is not None:
                copy.wait_event(freed[j])  # the run that read this set (batch k-2) is done
            q0 = 0
            for q1 in ends:
                r0, r1 = int(offsets[q0]), int(offsets[q1])
                for dst, src in zip(bufs[j], host_in):
                    dst[r0:r1].copy_(src[r0:r1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
                events.append(ev)
                q0 = q1
        return ends, events

    _t0 = time.perf_counter()
    host_pool = _PINNED_POOL  # shared by streams: pinned allocations are slow
    try:
        yield from _stream_loop(batches, cfg, prepare, h2d, bufs, freed, host_pool, comp, copy, _t0)
    finally:
        # a consumer may stop early: in-flight kernels and copies still use the
        # device buffers this generator owns, so drain both streams first
        copy.synchronize()
        comp.synchronize()


def _stream_loop(batches, cfg, prepare, h2d, bufs, freed, host_pool, comp, copy, _t0):
    import torch
    it = iter(batches)
    try:
        cur = prepare(next(it))
    except StopIteration:
        return
    k = 0
    cur_stage = h2d(0, cur[0], cur[1], staged=True)
    if _STREAM_DEBUG:
        print(f"[stream] first copies queued at {time.perf_counter() - _t0:.4f}", flush=True)
    pending = None  # (host results, done event, h2d bytes) of the previous batch
    while cur is not None:
        host_in, offsets, intrinsics, seeds = cur
        try:
            nxt = prepare(next(it))
        except StopIteration:
            nxt = None
        # batch k+1's copy is queued before batch k runs (its buffer set was
        # read by batch k-1, already finished) so it streams during the run
        nxt_stage = h2d(k + 1, nxt[0], nxt[1], staged=False) if nxt is not None else None
        N = int(offsets[-1])
        j = k % 2
        if _STREAM_DEBUG:
            print(f"[stream] batch {k}: launch run at {time.perf_counter() - _t0:.4f}", flush=True)
        out = ransac_pnp_device(bufs[j][0], bufs[j][1], bufs[j][2], offsets, intrinsics, seeds, cfg,
                                stages=cur_stage)
        if _STREAM_DEBUG:
            print(f"[stream] batch {k}: run returned at {time.perf_counter() - _t0:.4f}", flush=True)
        ev = torch.cuda.Event()
        ev.record(comp)
        freed[j] = ev
        # results D2H on the copy stream (overlaps the next run); batch k is
        # handed out once batch k+1 has been launched
        host_out = host_pool.get({key: (tuple(v.shape) if key != "flags" else (N,), v.dtype)
                                  for key, v in out.items()})
        with torch.cuda.stream(copy):
            copy.wait_event(ev)
            for key, v in out.items():
                v.record_stream(copy)
                host_out.tensors[key].copy_(v[:N] if key == "flags" else v, non_blocking=True)
            done = torch.cuda.Event()
            done.record(copy)
        h2d_bytes = sum(int(t.numel() * t.element_size()) for t in host_in)
        if _STREAM_DEBUG:
            print(f"[stream] batch {k}: D2H queued at {time.perf_counter() - _t0:.4f}", flush=True)
        if pending is not None:
            r = _stream_result(*pending)
            if _STREAM_DEBUG:
                print(f"[stream] batch {k - 1}: results ready at {time.perf_counter() - _t0:.4f}", flush=True)
            yield r
        pending = (host_out, done, h2d_bytes)
        cur, cur_stage = nxt, nxt_stage
        k += 1
    if pending is not None:
        yield _stream_result(*pending)


def _stream_result(host_out, done, h2d_bytes):
    done.synchronize()
    host = {key: v.numpy() for key, v in host_out.tensors.items()}
    host_out.hand_out(host.values())
    return host, h2d_bytes, sum(int(v.nbytes) for v in host.values())


class _PinnedPool:
    """Pinned host result buffers reused across the batches of a stream.

    A buffer set is reused only once every numpy array handed out from it has
    been released by the caller (weak references), so results stay valid for
    as long as they are referenced; a fresh pinned allocation (slow: it can
    cost tens of ms) is only made when no released set of the right shapes
    exists."""

    class _Set:
        def __init__(self, spec):
            import torch
            self.spec = spec
            self.tensors = {k: torch.empty(shape, dtype=dt, pin_memory=True) for k, (shape, dt) in spec.items()}
            self.refs = []

        def free(self):
            return all(r() is None for r in self.refs)

        def hand_out(self, arrays):
            import weakref
            self.refs = [weakref.ref(a) for a in arrays]

    def __init__(self):
        self.sets = []

    def get(self, spec):
        for st in self.sets:
            if st.spec == spec and st.free():
                st.refs = [lambda: True]  # busy until handed out
                return st
        st = _PinnedPool._Set(spec)
        st.refs = [lambda: True]
        self.sets.append(st)
        if len(self.sets) > 8:  # drop the oldest released sets beyond a small cache
            self.sets = [x for x in self.sets[:-8] if not x.free()] + self.sets[-8:]
        return st


_PINNED_POOL = _PinnedPool()


def _host_pipeline_chunks(host_in, offsets, intrinsics, seeds, cfg, chunk_queries, out, host_out, comp, copy, dev):
    """Separate estimator calls per chunk, double-buffered H2D / D2H on `copy`."""
    import torch
    Q = offsets.shape[0] - 1
    chunks = _host_chunks(Q, chunk_queries)
    max_rows = max(int(offsets[b] - offsets[a]) for a, b in chunks)
    bufs = [[torch.empty((max_rows,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev) for t in host_in]
            for _ in range(min(2, len(chunks)))]
    ev_in = [torch.cuda.Event() for _ in chunks]
    ev_done = [torch.cuda.Event() for _ in chunks]

    def h2d(k):
        a, b = chunks[k]
        r0, r1 = int(offsets[a]), int(offsets[b])
        with torch.cuda.stream(copy):
            if k >= 2:
                copy.wait_event(ev_done[k - 2])  # buffer k%2 was read by chunk k-2
            for dst, src in zip(bufs[k % 2], host_in):
                dst[: r1 - r0].copy_(src[r0:r1], non_blocking=True)
            ev_in[k].record(copy)

    copy.wait_stream(comp)
    h2d(0)
    for k, (a, b) in enumerate(chunks):
        r0, r1 = int(offsets[a]), int(offsets[b])
        if k + 1 < len(chunks):
            h2d(k + 1)
        comp.wait_event(ev_in[k])
        view = {key: (v[a:b] if key != "flags" else v[r0:r1]) for key, v in out.items()}
        d = [buf[: r1 - r0] for buf in bufs[k % 2]]
        ransac_pnp_device(d[0], d[1], d[2], offsets[a:b + 1] - offsets[a], intrinsics[a:b], seeds[a:b], cfg,
                          out=view)
        ev_done[k].record(comp)
        with torch.cuda.stream(copy):
            copy.wait_event(ev_done[k])
            for key, v in view.items():
                dst = host_out[key][a:b] if key != "flags" else host_out[key][r0:r1]
                dst.copy_(v, non_blocking=True)
    copy.synchronize()
    comp.wait_stream(copy)


def ransac_pnp_batch(queries, intrinsics, cfg: RansacConfig, seeds=None) -> list[PoseEstimate]:
    """Estimate many independent queries in one device-resident run.

    ``queries``: list of match sets (as ``ransac_pnp`` accepts);
    ``intrinsics``: one ``CameraIntrinsics`` or one per query; ``seeds``:
    per-query seeds (default ``cfg.seed`` for every query).
    """
    arrs = [_host_arrays(m) for m in queries]
    Q = len(arrs)
    if Q == 0:
        return []
    if isinstance(intrinsics, CameraIntrinsics) or not isinstance(intrinsics, (list, tuple)):
        intrinsics = [intrinsics] * Q
    if seeds is None:
        seeds = [cfg.seed] * Q
    offsets = np.zeros(Q + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([a[0].shape[0] for a in arrs])
    for i in range(Q):
        if offsets[i + 1] - offsets[i] < 3:
            raise UnderConstrainedError(f"need >= 3 matches, got {offsets[i + 1] - offsets[i]}")
    # one pinned staging buffer px | X | w and ONE host-to-device copy
    import torch
    _lib.context()  # fails loudly (VislocError) without a CUDA device / built library
    N = int(offsets[-1])
    h = torch.empty((6 * N,), dtype=torch.float64, pin_memory=True)
    hn = h.numpy()
    np.concatenate([a[0].reshape(-1) for a in arrs], out=hn[:2 * N])
    np.concatenate([a[1].reshape(-1) for a in arrs], out=hn[2 * N:5 * N])
    np.concatenate([a[2] for a in arrs], out=hn[5 * N:])
    d = h.cuda(non_blocking=True)
    px, X, w = d[:2 * N].view(N, 2), d[2 * N:5 * N].view(N, 3), d[5 * N:]
    out = ransac_pnp_device(px, X, w, offsets, intrinsics, seeds, cfg)
    return _estimates_from(out, offsets)


def ransac_pnp(matches, intr: CameraIntrinsics, cfg: RansacConfig) -> PoseEstimate:
    """Estimate a camera-from-world pose from weighted 2D-3D matches (posest.py:223)."""
    px, X, w = _host_arrays(matches)
    if px.shape[0] < 3:
        raise UnderConstrainedError(f"need >= 3 matches, got {px.shape[0]}")
    return ransac_pnp_batch([(px, X, w)], [intr], cfg, seeds=[cfg.seed])[0]


def msac_score(pose: Pose, matches, intr: CameraIntrinsics, tau: float):
    """Weighted MSAC cost and inlier flags (posest.py:160-175), fp64 on the GPU."""
    import torch
    px, X, w = _host_arrays(matches)
    n = px.shape[0]
    ctx = _lib.context()
    dpx, dX, dw = _to_device(px), _to_device(X), _to_device(w)
    flags = torch.empty((max(n, 1),), dtype=torch.uint8, device=dpx.device)
    q = np.ascontiguousarray(pose.q, dtype=np.float64)
    t = np.ascontiguousarray(pose.t, dtype=np.float64)
    cost = C.c_double()
    dp = C.POINTER(C.c_double)
    rc = _lib.lib().vl_msac_score(ctx.handle, q.ctypes.data_as(dp), t.ctypes.data_as(dp),
                                  dpx.data_ptr(), dX.data_ptr(), dw.data_ptr(), n, _intr_c(intr),
                                  float(tau), C.byref(cost), flags.data_ptr(), _lib.stream_ptr())
    ctx.check(rc, "vl_msac_score")
    return float(cost.value), flags[:n].cpu().numpy().astype(bool)


def score_hypotheses(Rs, ts, X, px, w, intr: CameraIntrinsics, tau: float, shape: int = 0) -> np.ndarray:
    """fp32 MSAC ranking costs of many hypotheses against one correspondence set
    (``_score_hypotheses``, posest.py:178-220), computed by the estimator's own
    k_score kernel.  Returns float64 like the reference (the values are fp32).
    ``shape`` selects the scoring tiles (0 single-query default, 1 fine, 2
    coarse); every shape gives the same bits."""
    import torch
    Rs = np.ascontiguousarray(Rs, dtype=np.float64).reshape(-1, 3, 3)
    ts = np.ascontiguousarray(ts, dtype=np.float64).reshape(-1, 3)
    px, X, w = _host_arrays((px, X, w))
    H, n = Rs.shape[0], px.shape[0]
    ctx = _lib.context()
    dR, dt = _to_device(Rs), _to_device(ts)
    dpx, dX, dw = _to_device(px), _to_device(X), _to_device(w)
    out = torch.empty((max(H, 1),), dtype=torch.float32, device=dpx.device)
    rc = _lib.lib().vl_score_hypotheses(ctx.handle, dR.data_ptr(), dt.data_ptr(), H, dpx.data_ptr(),
                                        dX.data_ptr(), dw.data_ptr(), n, _intr_c(intr), float(tau), int(shape),
                                        out.data_ptr(), _lib.stream_ptr())
    ctx.check(rc, "vl_score_hypotheses")
    return out[:H].cpu().numpy().astype(np.float64)
