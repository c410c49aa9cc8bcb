"""Probe: two query groups estimated concurrently on two streams (two contexts,
two host threads) vs one batched run — does the latency-bound fp64 work of one
group hide under the other's FP32 scoring?  GPU only:
    python tools/overlap_probe.py [Q] [groups]
"""
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2601_04185_b200 import _lib  # noqa: E402
from paper_2601_04185_b200.geometry import CameraIntrinsics  # noqa: E402
from paper_2601_04185_b200.posest import RansacConfig, ransac_pnp_device  # noqa: E402


def main():
    Q = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    wl = bench.WORKLOADS["c3"]
    n = wl["n"]
    qs = [bench.query_a(qi, n, wl["outlier"], wl["sigma"], 3000) for qi in range(Q)]
    d = [torch.from_numpy(np.concatenate([q[k] for q in qs])).cuda() for k in range(3)]
    offsets = np.arange(Q + 1, dtype=np.int64) * n
    intr = [CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * Q
    seeds = [bench.query_seed(qi, 3000) for qi in range(Q)]
    cfg = RansacConfig(max_iterations=wl["max_iterations"], miss_probability=wl["eta"])
    ref = ransac_pnp_device(d[0], d[1], d[2], offsets, intr, seeds, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        ransac_pnp_device(d[0], d[1], d[2], offsets, intr, seeds, cfg, out=ref)
    torch.cuda.synchronize()
    print(f"one run of {Q}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms")
    # G groups on G streams / contexts / host threads
    bounds = [Q * g // G for g in range(G + 1)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    ctxs = [_lib.Context(0) for _ in range(G)]
    outs = [None] * G

    def work_ctx(g, reps):
        a, b = bounds[g], bounds[g + 1]
        r0, r1 = int(offsets[a]), int(offsets[b])
        with torch.cuda.stream(streams[g]):
            for _ in range(reps):
                outs[g] = ransac_pnp_device(d[0][r0:r1], d[1][r0:r1], d[2][r0:r1], offsets[a:b + 1] - offsets[a],
                                            intr[a:b], seeds[a:b], cfg, ctx=ctxs[g])
    for g in range(G):
        work_ctx(g, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th = [threading.Thread(target=work_ctx, args=(g, 3)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    print(f"{G} concurrent groups: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms per {Q} queries")
    same = all(torch.equal(outs[g]["q"], ref["q"][bounds[g]:bounds[g + 1]]) for g in range(G))
    print("results equal to the single run:", same)


if __name__ == "__main__":
    main()
