"""Multi-process (gloo, world_size 2) checks of the query-sharding host logic."""

import os
import socket

import pytest

from paper_2601_04185_b200.dist import run_sharded, shard_indices, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_shard_indices_partition():
    for n in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            for mode in ("interleaved", "contiguous"):
                owned = [i for r in range(world) for i in shard_indices(n, r, world, mode)]
                assert sorted(owned) == list(range(n))
            assert shard_indices(n, world - 1, world, "interleaved") == list(range(world - 1, n, world))
    with pytest.raises(ValueError):
        shard_indices(4, 0, 2, "random")


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
    out_c = run_sharded(list(range(11)), lambda local: [-x for x in local], mode="contiguous")
    assert out_c == [-x for x in range(11)]
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
    assert res[0][2] == list(range(0, 11, 2)) and res[1][2] == list(range(1, 11, 2))  # interleaved


def test_bench_gpus_spawns_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself
    under torch.distributed.run: 2 ranks, one JSON line from rank 0 with
    n_gpus 2, interleaved shards covering the 1000-query job, a max-over-ranks
    time (VISLOC_BENCH_DRYRUN: the launcher and reductions only, on gloo)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["VISLOC_BENCH_DRYRUN"] = "1"
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2"], capture_output=True, text=True,
                       env=env, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["queries_total"] == 1000 and d["max_over_ranks"] == 2.0
