"""Timing probe of the host-buffer pipeline (ransac_pnp_host) on the C3 workload.

Prints raw pinned H2D bandwidth, device-only time per chunk size and the
end-to-end time of several chunk schedules.  GPU only:
    python tools/host_pipe.py [Q]
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2601_04185_b200 import posest  # noqa: E402
from paper_2601_04185_b200.geometry import CameraIntrinsics  # noqa: E402
from paper_2601_04185_b200.posest import RansacConfig, ransac_pnp_device, ransac_pnp_host  # noqa: E402


def ev_time(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


def main():
    Q = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    wl = bench.WORKLOADS["c3"]
    n = wl["n"]
    seed0 = 3000
    qs = [bench.query_a(qi, n, wl["outlier"], wl["sigma"], seed0) for qi in range(Q)]
    px_h = torch.from_numpy(np.concatenate([q[0] for q in qs])).pin_memory()
    X_h = torch.from_numpy(np.concatenate([q[1] for q in qs])).pin_memory()
    w_h = torch.from_numpy(np.concatenate([q[2] for q in qs])).pin_memory()
    offsets = np.arange(Q + 1, dtype=np.int64) * n
    intr = [CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * Q
    seeds = [bench.query_seed(qi, seed0) for qi in range(Q)]
    cfg = RansacConfig(max_iterations=wl["max_iterations"], miss_probability=wl["eta"])
    px_d, X_d, w_d = px_h.cuda(), X_h.cuda(), w_h.cuda()

    def h2d():
        px_d.copy_(px_h, non_blocking=True)
        X_d.copy_(X_h, non_blocking=True)
        w_d.copy_(w_h, non_blocking=True)
    ms, wall = ev_time(h2d)
    nb = (px_h.numel() + X_h.numel() + w_h.numel()) * 8
    print(f"H2D {nb / 1e9:.2f} GB: {ms:.2f} ms = {nb / ms / 1e6:.1f} GB/s")

    for qq in (63, 126, 252, 559, Q):
        o = offsets[: qq + 1]
        n_r = int(o[-1])
        ms, wall = ev_time(lambda: ransac_pnp_device(px_d[:n_r], X_d[:n_r], w_d[:n_r], o, intr[:qq], seeds[:qq], cfg))
        print(f"device Q={qq:5d}: {ms:8.2f} ms (wall {wall:8.2f})")

    for sched in (63, 256, Q):
        ms, wall = ev_time(lambda: ransac_pnp_host(px_h, X_h, w_h, offsets, intr, seeds, cfg, chunk_queries=sched))
        print(f"host chunks={posest._host_chunks(Q, sched)[:6]}: {ms:8.2f} ms (wall {wall:8.2f})")
    f = Q / 1000
    for ends in (posest._stage_schedule(Q), [int(f * e) for e in (63, 189, 441, 1000)],
                 [int(f * e) for e in (125, 375, 1000)], [int(f * e) for e in (125, 250, 500, 1000)],
                 [int(f * e) for e in (250, 1000)], [int(f * e) for e in (100, 200, 300, 400, 500, 600, 700, 800,
                                                                          900, 1000)]):
        ms, wall = ev_time(lambda: ransac_pnp_host(px_h, X_h, w_h, offsets, intr, seeds, cfg, stage_ends=ends))
        print(f"staged ends={ends}: {ms:8.2f} ms (wall {wall:8.2f})")


if __name__ == "__main__" and len(sys.argv) <= 2:
    main()


def profile_compare():
    """Stage breakdown: device-resident run vs staged host run (C3)."""
    from paper_2601_04185_b200 import _lib
    Q = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
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
    ctx = _lib.context()
    for name, fn in (("device", lambda: ransac_pnp_device(px_d, X_d, w_d, offsets, intr, seeds, cfg)),
                     ("staged", lambda: ransac_pnp_host(px_h, X_h, w_h, offsets, intr, seeds, cfg))):
        fn()
        torch.cuda.synchronize()
        ctx.profile(True)
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        prof = ctx.profile_read()
        ctx.profile(False)
        print(name, f"wall {wall:.2f} ms", {k: (round(v[0], 2), v[1]) for k, v in prof.items() if v[1]})


if __name__ == "__main__" and len(sys.argv) > 2:
    profile_compare()
