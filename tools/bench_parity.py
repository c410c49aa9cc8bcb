"""Parity of the benchmarked workloads themselves against the CPU oracle (tools only).

    python tools/bench_parity.py [N] [c3|c3p|c3a|c5|all]

Runs the GPU estimator on the bench's full batch — C3 / C3p (pruned) / C3a: the 1000
generator-A queries of `bench.py` with its seeds; C5: the 256 lifted queries
(8-bit depth, IMLC-style f32 fields) through `LiftPlan` exactly as the bench
times them — and compares the first N queries of that batch with the
oracle (`oracle/`, bit-exact restatement of the reference, run on all host
cores): iterations, LO calls, convergence, pose (0.01 deg / 1e-4 rel. t) and
inlier masks (identical except points within 1e-6 px of tau under the GPU or
oracle pose).  Prints one JSON line per workload.
"""
import json
import multiprocessing as mp
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]


def _oracle_a(job):
    qi, wl = job
    os.environ["OMP_NUM_THREADS"] = "1"
    from bench import query_a, query_seed
    from oracle.posest import Config, ransac
    px, X, w = query_a(qi, wl["n"], wl["outlier"], wl["sigma"], 3000)
    o = ransac(px, X, w, (700.0, 700.0, 350.0, 350.0),
               Config(seed=query_seed(qi, 3000), max_iterations=wl["max_iterations"], miss_probability=wl["eta"]))
    return o


def _oracle_c5(job):
    qi, wl = job
    os.environ["OMP_NUM_THREADS"] = "1"
    from bench import LIFT_SEED, query_seed
    from oracle import lift as ol
    from oracle.geometry import q2R
    from oracle.posest import Config, ransac
    from synth_inputs import lifted_scene
    vmap, jobs, dc = lifted_scene(wl["K"], wl["queries"], wl["g"], seed=LIFT_SEED, depth_kind=wl["depth"],
                                  only=[qi], fields="f32")
    pxs, Xs, ws = [], [], []
    for e in sorted(vmap.entries, key=lambda e: e.id):
        fp = jobs[0].fields[e.id]
        q = e.qdepth
        vals, valid = ol.dequantize(q.codes, q.d_min, q.d_max, q.levels)
        f1 = (fp.db_to_query.targets, fp.db_to_query.confidence, fp.db_to_query.scale_x, fp.db_to_query.scale_y)
        f2 = (fp.query_to_db.targets, fp.query_to_db.confidence, fp.query_to_db.scale_x, fp.query_to_db.scale_y)
        I = e.intrinsics
        px, X, w = ol.lift(f1, f2, vals, valid, (I.fx, I.fy, I.cx, I.cy), (I.width, I.height), q2R(e.pose.q),
                           e.pose.t, 0.05)
        pxs.append(px)
        Xs.append(X)
        ws.append(w)
    px, X, w = np.concatenate(pxs), np.concatenate(Xs), np.concatenate(ws)
    I = jobs[0].intrinsics
    o = ransac(px, X, w, (I.fx, I.fy, I.cx, I.cy),
               Config(seed=query_seed(qi, LIFT_SEED), max_iterations=wl["max_iterations"], miss_probability=wl["eta"]))
    return o, px, X, (I.fx, I.fy, I.cx, I.cy)


def _compare(name, gpu, ref, data):
    """gpu: list of (q, t, flags, iters, lo, conv); ref: oracle Results; data: (px, X, intr) per query."""
    from oracle import geometry as og
    from parity_util import near_threshold
    st = dict(workload=name, queries=len(ref), same_iterations=0, same_lo_calls=0, same_converged=0,
              pose_within_tol=0, masks_identical_or_near_tau=0, masks_bit_identical=0, max_rot_deg=0.0,
              max_rel_t=0.0, mask_diff_points=0)
    for (q, t, flags, iters, lo, conv), o, (px, X, intr) in zip(gpu, ref, data):
        st["same_iterations"] += int(iters == o.iterations)
        st["same_lo_calls"] += int(lo == o.lo_calls)
        st["same_converged"] += int(bool(conv) == bool(o.converged))
        rot = og.rot_err_deg(q, o.q)
        rel = float(np.linalg.norm(t - o.t) / max(np.linalg.norm(o.t), 1e-12))
        st["max_rot_deg"] = max(st["max_rot_deg"], rot)
        st["max_rel_t"] = max(st["max_rel_t"], rel)
        st["pose_within_tol"] += int(rot < 0.01 and rel < 1e-4)
        diff = flags != o.inlier_flags
        st["mask_diff_points"] += int(diff.sum())
        st["masks_bit_identical"] += int(not diff.any())
        if diff.any():
            amb = near_threshold(q, t, px, X, intr, 12.0) | near_threshold(o.q, o.t, px, X, intr, 12.0)
            st["masks_identical_or_near_tau"] += int(not (diff & ~amb).any())
        else:
            st["masks_identical_or_near_tau"] += 1
    return st


def run_a(name, N):
    import torch
    from bench import WORKLOADS, query_a, query_seed
    from paper_2601_04185_b200.geometry import CameraIntrinsics
    from paper_2601_04185_b200.posest import RansacConfig, ransac_pnp_device
    wl = WORKLOADS[name]
    Q, n = wl["queries"], wl["n"]
    from paper_2601_04185_b200 import _lib
    _lib.context().set_pruning(bool(wl.get("prune", True)))  # as bench.py runs the workload
    with mp.get_context("spawn").Pool(len(os.sched_getaffinity(0))) as pool:
        ref_async = pool.map_async(_oracle_a, [(qi, wl) for qi in range(N)], chunksize=1)
        qs = [query_a(qi, n, wl["outlier"], wl["sigma"], 3000) for qi in range(Q)]
        px = torch.from_numpy(np.concatenate([a[0] for a in qs])).cuda()
        X = torch.from_numpy(np.concatenate([a[1] for a in qs])).cuda()
        w = torch.from_numpy(np.concatenate([a[2] for a in qs])).cuda()
        off = np.arange(Q + 1, dtype=np.int64) * n
        intr = [CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * Q
        out = ransac_pnp_device(px, X, w, off, intr, [query_seed(qi, 3000) for qi in range(Q)],
                                RansacConfig(max_iterations=wl["max_iterations"], miss_probability=wl["eta"]))
        o = {k: v.cpu().numpy() for k, v in out.items()}
        ref = ref_async.get()
    gpu = [(o["q"][i], o["t"][i], o["flags"][i * n:(i + 1) * n].astype(bool), int(o["iterations"][i]),
            int(o["stats"][i, 0]), int(o["converged"][i])) for i in range(N)]
    data = [(qs[i][0], qs[i][1], (700.0, 700.0, 350.0, 350.0)) for i in range(N)]
    return _compare(name, gpu, ref, data)


def run_c5(N):
    from bench import LIFT_SEED, LIFT_WORKLOADS, query_seed
    from paper_2601_04185_b200.localizer import LiftPlan
    from paper_2601_04185_b200.posest import RansacConfig
    from synth_inputs import lifted_scene
    wl = LIFT_WORKLOADS["c5"]
    with mp.get_context("spawn").Pool(len(os.sched_getaffinity(0))) as pool:
        ref_async = pool.map_async(_oracle_c5, [(qi, wl) for qi in range(N)], chunksize=1)
        vmap, jobs, dc = lifted_scene(wl["K"], wl["queries"], wl["g"], seed=LIFT_SEED, depth_kind=wl["depth"],
                                      fields="f32")
        plan = LiftPlan(jobs, vmap, depth_cache=dc)
        cfg = RansacConfig(max_iterations=wl["max_iterations"], miss_probability=wl["eta"])
        ests = plan.localize(cfg, [query_seed(qi, LIFT_SEED) for qi in range(len(jobs))])
        res = ref_async.get()
    gpu = [(e.pose.q, e.pose.t, e.inlier_flags, e.iterations, e.stats["lo_calls"], e.converged) for e in ests[:N]]
    ref = [r[0] for r in res]
    data = [(r[1], r[2], r[3]) for r in res]
    return _compare("c5", gpu, ref, data)


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    which = sys.argv[2] if len(sys.argv) > 2 else "all"
    for name in (["c3", "c3p", "c3a", "c5"] if which == "all" else [which]):
        st = run_c5(N) if name == "c5" else run_a(name, N)
        print(json.dumps(st), flush=True)


if __name__ == "__main__":
    main()
