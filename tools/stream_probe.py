"""Timing probe of the serving stream (ransac_pnp_stream) on the C3 workload (tools only).

Device-resident runs vs device runs with a concurrent 2.4 GB H2D on a side
stream vs the stream itself (per-batch wall times).  GPU only:
    python tools/stream_probe.py [Q] [batches]
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2601_04185_b200.geometry import CameraIntrinsics  # noqa: E402
from paper_2601_04185_b200.posest import RansacConfig, ransac_pnp_device, ransac_pnp_stream  # noqa: E402


def main():
    Q = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    wl = bench.WORKLOADS["c3"]
    qs = [bench.query_a(qi, wl["n"], wl["outlier"], wl["sigma"], 3000) for qi in range(Q)]
    px_h = torch.from_numpy(np.concatenate([q[0] for q in qs])).pin_memory()
    X_h = torch.from_numpy(np.concatenate([q[1] for q in qs])).pin_memory()
    w_h = torch.from_numpy(np.concatenate([q[2] for q in qs])).pin_memory()
    offsets = np.arange(Q + 1, dtype=np.int64) * wl["n"]
    intr = [CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * Q
    seeds = [bench.query_seed(qi, 3000) for qi in range(Q)]
    cfg = RansacConfig(max_iterations=wl["max_iterations"], miss_probability=wl["eta"])
    px_d, X_d, w_d = px_h.cuda(), X_h.cuda(), w_h.cuda()
    out = ransac_pnp_device(px_d, X_d, w_d, offsets, intr, seeds, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        ransac_pnp_device(px_d, X_d, w_d, offsets, intr, seeds, cfg, out=out)
    torch.cuda.synchronize()
    print(f"device-resident: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms/batch")
    # same, with a concurrent H2D of the whole batch on a side stream
    side = torch.cuda.Stream()
    bufs = [torch.empty_like(px_d), torch.empty_like(X_d), torch.empty_like(w_d)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        with torch.cuda.stream(side):
            for d, h in zip(bufs, (px_h, X_h, w_h)):
                d.copy_(h, non_blocking=True)
        ransac_pnp_device(px_d, X_d, w_d, offsets, intr, seeds, cfg, out=out)
    torch.cuda.synchronize()
    print(f"device-resident + concurrent H2D: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms/batch")
    batch = (px_h, X_h, w_h, offsets, intr, seeds)
    for res in ransac_pnp_stream([batch] * 3, cfg):
        del res
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    last = t0
    for k, res in enumerate(ransac_pnp_stream([batch] * nb, cfg)):
        del res
        now = time.perf_counter()
        print(f"  stream batch {k}: +{(now - last) * 1e3:.2f} ms")
        last = now
    torch.cuda.synchronize()
    print(f"stream: {(time.perf_counter() - t0) / nb * 1e3:.2f} ms/batch over {nb}")


if __name__ == "__main__":
    main()
