"""ransac_pnp_split through torch.distributed with 2 real processes (gloo
all-reduce of the CUDA partial-cost buffer; both ranks share the one GPU —
their kernels never wait on each other, the exchange is host-side)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q, mode="sum"):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path[:0] = [str(root), str(root / "tests")]
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    import paper_2601_04185_b200 as vl
    from paper_2601_04185_b200.dist import ransac_pnp_split
    from synth_inputs import matches_a
    px, X, w, _ = matches_a(5000, 0.6, 1.0, seed=31)
    intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
    cfg = vl.RansacConfig(seed=8, max_iterations=3000, miss_probability=1e-300)
    e = ransac_pnp_split((px, X, w), intr, cfg, mode=mode)
    if mode == "sum":
        ref = vl.ransac_pnp((px, X, w), intr, cfg)
    else:  # the approximate variant must not depend on the split size
        singles = [dist.new_group([0]), dist.new_group([1])]  # collective: every rank creates both
        ref = ransac_pnp_split((px, X, w), intr, cfg, group=singles[rank], mode=mode)
    q.put((rank, np.array_equal(e.pose.q, ref.pose.q) and np.array_equal(e.inlier_flags, ref.inlier_flags),
           e.pose.q.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["sum", "argmin"])
def test_split_two_processes(mode):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, port, q, mode)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0][1] and res[1][1]
    assert res[0][2] == res[1][2]
