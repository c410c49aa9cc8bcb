"""Query sharding across GPUs (one process per GPU, torch.distributed plumbing).

Queries are independent (reference SPEC: per-query determinism, no shared
state), so the multi-GPU path partitions whole queries into contiguous
shards with **no collective on the data path**; each rank runs the batched
device estimator on its shard and results are gathered only for reporting
(`all_gather_object` / a scalar max for timing).  Sharding never changes a
query's result: each query keeps its own seed.
"""

from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def run_sharded(items, fn, group=None):
    """Apply `fn(local_items) -> list` on this rank's shard; every rank gets all
    results in the original order (gathered as Python objects)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return list(fn(list(items)))
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(len(items), rank, world)
    local = list(fn(list(items[lo:hi])))
    if len(local) != hi - lo:
        raise RuntimeError("fn must return one result per item")
    gathered = [None] * world
    dist.all_gather_object(gathered, local, group=group)
    out = []
    for part in gathered:
        out.extend(part)
    return out


def localize_sharded(jobs, vmap, cfg, seeds=None, group=None, **kw):
    """``localize_batch`` over all ranks' GPUs (each rank: its own shard, its own device)."""
    from .localizer import localize_batch
    jobs = list(jobs)
    seeds = list(seeds) if seeds is not None else [cfg.seed] * len(jobs)
    pairs = list(zip(jobs, seeds))

    def fn(local):
        if not local:
            return []
        return localize_batch([j for j, _ in local], vmap, cfg, seeds=[s for _, s in local], **kw)

    return run_sharded(pairs, fn, group)


def ransac_pnp_sharded(queries, intrinsics, cfg, seeds=None, group=None):
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

    return run_sharded(triples, fn, group)
