"""Small fixed workload for ncu captures: one batched ransac_pnp call.

    python tools/prof_case.py --queries 100 --n 50000 --iters 2000 [--reps 2]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--queries", type=int, default=100)
    ap.add_argument("--n", type=int, default=50_000)
    ap.add_argument("--iters", type=int, default=2000)
    ap.add_argument("--outlier", type=float, default=0.7)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch
    from bench import query_a, query_seed
    from paper_2601_04185_b200.geometry import CameraIntrinsics
    from paper_2601_04185_b200.posest import RansacConfig, ransac_pnp_device
    qs = [query_a(i, a.n, a.outlier, 1.0, 3000) for i in range(a.queries)]
    px = torch.from_numpy(np.concatenate([q[0] for q in qs])).cuda()
    X = torch.from_numpy(np.concatenate([q[1] for q in qs])).cuda()
    w = torch.from_numpy(np.concatenate([q[2] for q in qs])).cuda()
    off = np.arange(a.queries + 1, dtype=np.int64) * a.n
    intr = [CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * a.queries
    seeds = [query_seed(i, 3000) for i in range(a.queries)]
    cfg = RansacConfig(max_iterations=a.iters, miss_probability=1e-300)
    out = None
    for _ in range(a.reps):
        out = ransac_pnp_device(px, X, w, off, intr, seeds, cfg, out=out)
    torch.cuda.synchronize()
    print("ok", int(out["converged"].sum().item()), "/", a.queries)


if __name__ == "__main__":
    main()
