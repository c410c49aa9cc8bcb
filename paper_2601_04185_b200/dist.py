"""Query sharding across GPUs (one process per GPU, torch.distributed plumbing).

Queries are independent (reference SPEC: per-query determinism, no shared
state), so the multi-GPU path partitions whole queries across ranks with
**no collective on the data path**; each rank runs the batched device
estimator on its shard and results are gathered only for reporting
(`all_gather_object` / a scalar max for timing).  Sharding never changes a
query's result: each query keeps its own seed.

Assignment is interleaved by default (rank r owns queries r, r + G, r + 2G,
...): adaptive stopping makes per-query cost uneven, and neighbouring
queries of a real batch (one image sequence) tend to be alike, so blocks
would load some ranks with all the hard queries.  Contiguous
blocks (`shard_range`) remain available.
"""

from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_indices(n: int, rank: int, world: int, mode: str = "interleaved") -> list[int]:
    """Indices of the n items owned by `rank`: ``interleaved`` (r, r+G, ...) or
    ``contiguous`` (the `shard_range` block).  Every item has exactly one owner."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if mode == "interleaved":
        return list(range(rank, n, world))
    if mode == "contiguous":
        lo, hi = shard_range(n, rank, world)
        return list(range(lo, hi))
    raise ValueError(f"mode must be 'interleaved' or 'contiguous', got {mode!r}")


def run_sharded(items, fn, group=None, mode: str = "interleaved"):
    """Apply `fn(local_items) -> list` on this rank's shard; every rank gets all
    results in the original order (gathered as Python objects)."""
    import torch.distributed as dist
    items = list(items)
    if not (dist.is_available() and dist.is_initialized()):
        return list(fn(items))
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = shard_indices(len(items), rank, world, mode)
    local = list(fn([items[i] for i in mine]))
    if len(local) != len(mine):
        raise RuntimeError("fn must return one result per item")
    gathered = [None] * world
    dist.all_gather_object(gathered, local, group=group)
    out = [None] * len(items)
    for r, part in enumerate(gathered):
        for i, v in zip(shard_indices(len(items), r, world, mode), part):
            out[i] = v
    return out


class SplitRun:
    """One rank's side of the hypothesis-split estimator.

    Drives the C ABI stepwise driver (``vl_ransac_begin`` / ``step_score`` /
    ``step_finish`` / ``end``) for queries whose matches are already on this
    rank's device.  The caller reduces ``self.partial`` (SUM) across ranks
    between ``score()`` and ``finish()``.
    """

    def __init__(self, ctx, px, X, w, offsets, intrinsics, seeds, cfg, rank: int, size: int):
        import ctypes as C

        import numpy as np
        import torch

        from . import _lib
        from .posest import _cfg_c, _intr_c
        self.ctx, self.L = ctx, _lib.lib()
        self._keep = (px, X, w)
        offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
        Q = offsets.shape[0] - 1
        self.offsets, self.Q = offsets, Q
        self._intr = (_lib.Intrinsics * Q)(*[_intr_c(i) for i in intrinsics])
        self._rng = (_lib.PCG64State * Q)(*[_lib.pcg64_state(int(s)) for s in seeds])
        a = _lib.RansacArgs()
        a.num_queries = Q
        a.offsets = offsets.ctypes.data_as(C.POINTER(C.c_int64))
        a.intr, a.rng = self._intr, self._rng
        a.px, a.X, a.w = px.data_ptr(), X.data_ptr(), w.data_ptr()
        a.cfg = _cfg_c(cfg)
        self._args = a
        ctx.check(self.L.vl_ransac_begin(ctx.handle, C.byref(a), rank, size, _lib.stream_ptr()), "vl_ransac_begin")
        nb = C.c_int64()
        ctx.check(self.L.vl_ransac_partial_bytes(ctx.handle, C.byref(nb)), "vl_ransac_partial_bytes")
        self.partial = torch.empty((nb.value // 4,), dtype=torch.float32, device=px.device)
        self.nactive = Q

    def score(self):
        from . import _lib
        self.ctx.check(self.L.vl_ransac_step_score(self.ctx.handle, self.partial.data_ptr(), _lib.stream_ptr()),
                       "vl_ransac_step_score")

    def argmin(self):
        """Packed (score, index) keys of this rank's owned hypotheses -> ``self.keys`` (int64 [Q])."""
        import torch

        from . import _lib
        if getattr(self, "keys", None) is None:
            self.keys = torch.empty((self.Q,), dtype=torch.int64, device=self.partial.device)
        self.ctx.check(self.L.vl_ransac_step_argmin(self.ctx.handle, self.keys.data_ptr(), _lib.stream_ptr()),
                       "vl_ransac_step_argmin")

    def finish_argmin(self) -> int:
        import ctypes as C

        from . import _lib
        n = C.c_int32()
        self.ctx.check(self.L.vl_ransac_step_finish_argmin(self.ctx.handle, self.keys.data_ptr(), C.byref(n),
                                                           _lib.stream_ptr()), "vl_ransac_step_finish_argmin")
        self.nactive = int(n.value)
        return self.nactive

    def finish(self) -> int:
        import ctypes as C

        from . import _lib
        n = C.c_int32()
        self.ctx.check(self.L.vl_ransac_step_finish(self.ctx.handle, self.partial.data_ptr(), C.byref(n),
                                                    _lib.stream_ptr()), "vl_ransac_step_finish")
        self.nactive = int(n.value)
        return self.nactive

    def end(self):
        import ctypes as C

        import torch

        from . import _lib
        from .posest import _estimates_from
        dev = self.partial.device
        N = int(self.offsets[-1])
        Q = self.Q
        out = {"q": torch.empty((Q, 4), dtype=torch.float64, device=dev),
               "t": torch.empty((Q, 3), dtype=torch.float64, device=dev),
               "flags": torch.empty((max(N, 1),), dtype=torch.uint8, device=dev),
               "count": torch.empty((Q,), dtype=torch.int64, device=dev),
               "score": torch.empty((Q,), dtype=torch.float64, device=dev),
               "iterations": torch.empty((Q,), dtype=torch.int64, device=dev),
               "converged": torch.empty((Q,), dtype=torch.int32, device=dev),
               "stats": torch.empty((Q, 4), dtype=torch.int64, device=dev)}
        o = _lib.RansacOut()
        o.q, o.t, o.inlier_flags = out["q"].data_ptr(), out["t"].data_ptr(), out["flags"].data_ptr()
        o.inlier_count, o.score = out["count"].data_ptr(), out["score"].data_ptr()
        o.iterations, o.converged = out["iterations"].data_ptr(), out["converged"].data_ptr()
        o.stats = out["stats"].data_ptr()
        self.ctx.check(self.L.vl_ransac_end(self.ctx.handle, C.byref(o), _lib.stream_ptr()), "vl_ransac_end")
        out["flags"] = out["flags"][:N]
        return _estimates_from(out, self.offsets)


def ransac_pnp_split(matches, intr, cfg, group=None, mode: str = "sum"):
    """One query's hypotheses split across the ranks of `group` (one GPU each).

    Every rank passes the same matches and config.  ``mode="sum"`` (default):
    per round, one NCCL SUM all-reduce of the partial-cost buffer (SURVEY §8e
    "exact reference semantics" variant: the full cost vector, so the ordered
    first-better scan is unchanged) — the same PoseEstimate on every rank,
    bit-identical to ``ransac_pnp``.  ``mode="argmin"``: BASELINE's packed
    (score, index) variant — one MIN all-reduce of an 8-byte key per query
    per round; the scan then sees only the batch's best hypothesis (at most
    one LO per round), an APPROXIMATION of the reference's ordered chain that
    is identical on every rank and for every split size.
    """
    if mode not in ("sum", "argmin"):
        raise ValueError(f"mode must be 'sum' or 'argmin', got {mode!r}")
    import torch
    import torch.distributed as dist

    from . import _lib
    from .posest import UnderConstrainedError, _host_arrays, _to_device
    distributed = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if distributed else 0
    world = dist.get_world_size(group) if distributed else 1
    px, X, w = _host_arrays(matches)
    if px.shape[0] < 3:
        raise UnderConstrainedError(f"need >= 3 matches, got {px.shape[0]}")
    ctx = _lib.context()
    dpx, dX, dw = _to_device(px), _to_device(X), _to_device(w)
    run = SplitRun(ctx, dpx, dX, dw, [0, px.shape[0]], [intr], [cfg.seed], cfg, rank, world)
    while run.nactive > 0:
        run.score()
        if mode == "argmin":
            run.argmin()
            if world > 1:
                dist.all_reduce(run.keys, op=dist.ReduceOp.MIN, group=group)
            run.finish_argmin()
            continue
        if world > 1:
            dist.all_reduce(run.partial, op=dist.ReduceOp.SUM, group=group)
        run.finish()
    torch.cuda.current_stream().synchronize()
    return run.end()[0]


def localize_sharded(jobs, vmap, cfg, seeds=None, group=None, mode: str = "interleaved", **kw):
    """``localize_batch`` over all ranks' GPUs (each rank: its own shard, its own device)."""
    from .localizer import localize_batch
    jobs = list(jobs)
    seeds = list(seeds) if seeds is not None else [cfg.seed] * len(jobs)
    pairs = list(zip(jobs, seeds))

    def fn(local):
        if not local:
            return []
        return localize_batch([j for j, _ in local], vmap, cfg, seeds=[s for _, s in local], **kw)

    return run_sharded(pairs, fn, group, mode)


def ransac_pnp_sharded(queries, intrinsics, cfg, seeds=None, group=None, mode: str = "interleaved"):
    """``ransac_pnp_batch`` over all ranks' GPUs."""
    from .posest import ransac_pnp_batch
    queries = list(queries)
    if not isinstance(intrinsics, (list, tuple)):
        intrinsics = [intrinsics] * len(queries)
    seeds = list(seeds) if seeds is not None else [cfg.seed] * len(queries)
    triples = list(zip(queries, intrinsics, seeds))

    def fn(local):
        if not local:
            return []
        return ransac_pnp_batch([q for q, _, _ in local], [i for _, i, _ in local], cfg,
                                seeds=[s for _, _, s in local])

    return run_sharded(triples, fn, group, mode)
