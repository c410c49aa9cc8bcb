"""Multi-process (gloo, world_size 2) checks of the query-sharding host logic."""

import os
import socket

import pytest

from paper_2601_04185_b200.dist import run_sharded, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seen = []

    def fn(local):
        seen.extend(local)
        return [x * x for x in local]

    out = run_sharded(list(range(11)), fn)
    # timing reduction used by bench.py: max over ranks
    import torch
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, out, seen, float(t.item())))
    dist.destroy_process_group()


def test_run_sharded_gloo_world2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out, seen, tmax in res:
        assert out == [x * x for x in range(11)]
        assert tmax == 2.0
    assert res[0][2] == list(range(0, 6)) and res[1][2] == list(range(6, 11))
