#!/usr/bin/env python
"""Benchmark of the B200 LO-RANSAC PnP hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c3a|c1|c4|c2|c5|c5h|map]
                    [--impl ours|reference] [--no-configs]

One *step* = one complete batched ``ransac_pnp`` over the workload's
queries (sampling, P3P, fp32 scoring, LO, adaptive stop, final Cauchy
refinement) with inputs resident in HBM.  Default workload is BASELINE
config C3 ("Aachen-style batch": 1000 queries x 50k correspondences per GPU,
30% inliers, sigma 1 px) in fixed-iteration mode (10k minimal samples per
query, eta = 1e-300) so every query does the same, BASELINE-named amount of
work.  ``value`` = hypothesis x correspondence evaluations / s over the
whole job; ``e2e`` = the same through the host-buffer API (H2D of the packed
matches + D2H of poses/masks inside the timed region).

Multi-GPU: ``--gpus N`` without a torchrun environment re-launches itself
under ``torch.distributed.run`` (N ranks, one per GPU, NCCL, 127.0.0.1).
Queries shard with no collective.  ``value`` is weak scaling (1000 queries
per GPU); the line's ``strong`` object times the literal C3 batch of 1000
queries split across the N ranks (interleaved assignment, dist.shard_indices).

At N = 1 the default line also carries ``configs``: C3a (the same batch with
the adaptive default stop, whose serving e2e is PCIe-bound), BASELINE C1
(single query through the drop-in ``ransac_pnp``), C4 (low inlier ratio,
LO-heavy) and C5 (8-bit compressed map: GPU lift + estimator, lift HBM
roofline), each with its own value / e2e / roofline / cpu_baseline.

``--impl reference`` times the CPU reference arm: the oracle port of the
reference algorithm (``oracle/``, bit-identical to visloc on the golden
vectors) over all host cores on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

FLOP_PER_EVAL = 30  # literal count of posest.py:203-219

WORKLOADS = {
    "c3": dict(name="C3 Aachen-style batch: 1000 queries x 50k corrs per GPU, eps=0.3, sigma=1px, "
                    "fixed 10k minimal samples/query (eta=1e-300)",
               queries=1000, n=50_000, outlier=0.7, sigma=1.0, max_iterations=10_000, eta=1e-300,
               cpu_queries_per_core=2, prune=False),
    # the same batch with exact scoring pruning (vl_set_scoring_pruning): hypotheses whose fp32
    # prefix sum already reaches the best cost are not scored to the end; outputs identical, `value`
    # counts the reference's nominal evaluations (the roofline counts the executed ones)
    "c3p": dict(name="C3 Aachen-style batch: 1000 queries x 50k corrs per GPU, eps=0.3, sigma=1px, "
                     "fixed 10k minimal samples/query (eta=1e-300), exact scoring pruning",
                queries=1000, n=50_000, outlier=0.7, sigma=1.0, max_iterations=10_000, eta=1e-300,
                cpu_queries_per_core=2, prune=True),
    "c3a": dict(name="C3 Aachen-style batch, adaptive stop (eta=1e-4): 1000 queries x 50k corrs per GPU, "
                     "eps=0.3, sigma=1px",
                queries=1000, n=50_000, outlier=0.7, sigma=1.0, max_iterations=100_000, eta=1e-4,
                cpu_queries_per_core=2),
    "c1": dict(name="C1 single query: 2k corrs, eps=0.3, sigma=1px, fixed 10k minimal samples",
               queries=1, n=2_000, outlier=0.7, sigma=1.0, max_iterations=10_000, eta=1e-300,
               cpu_queries_per_core=1),
    "c4": dict(name="C4 low inlier ratio: 10k corrs, eps=0.05, 100k minimal samples (LO-heavy)",
               queries=1, n=10_000, outlier=0.95, sigma=1.0, max_iterations=100_000, eta=1e-300,
               cpu_queries_per_core=1, cpu_max_iterations=20_000),
}


LIFT_WORKLOADS = {
    "c2": dict(name="C2 single query, dense-matcher scale: K=20 db images x 83x83 bidirectional fields "
                    "(~226k lifted corrs), f32 depth lift, fixed 10k minimal samples",
               K=20, g=83, queries=1, depth="f32", max_iterations=10_000, eta=1e-300, cpu_queries_per_core=0.0625),
    "c5": dict(name="C5 compressed map: 8-bit log-quantised depth decode + lift, K=10 x 117x117 fields "
                    "(~20k lifted/entry), 256 queries, default adaptive config",
               K=10, g=117, queries=256, depth="u8", max_iterations=100_000, eta=1e-4, cpu_queries_per_core=2),
    "c5h": dict(name="C5 compressed map (fp16 depth variant): K=10 x 117x117 fields, 256 queries, "
                     "default adaptive config",
                K=10, g=117, queries=256, depth="f16", max_iterations=100_000, eta=1e-4, cpu_queries_per_core=2),
}
LIFT_SEED = 77

MAP_WORKLOADS = {
    "map": dict(name="Mapping (SURVEY 8f rows 3-4): dense depth triangulation + 8-bit log quantisation of "
                     "64 db images x 20 covisible views x 83x83 f32 fields, default TriangulationConfig",
                E=64, V=20, g=83, cpu_maps_per_core=1),
}
MAP_SEED = 5
VOTE_FLOP = 27  # fp64 ops of one (hypothesis, view) angular vote test


def _cpu_map_worker(job):
    """Oracle port of build_depth_map + quantize_depth for one entry of the mapping workload."""
    i, wl, seed0 = job
    from oracle import depthbuild as od
    from oracle import mapstore as om
    from synth_inputs import mapping_scene
    (e, cv, fl), = mapping_scene(wl["E"], wl["V"], wl["g"], seed=seed0, only=[i])
    I = e.intrinsics
    irow = lambda c: [c.intrinsics.fx, c.intrinsics.fy, c.intrinsics.cx, c.intrinsics.cy,  # noqa: E731
                      c.intrinsics.width, c.intrinsics.height]
    t0 = time.perf_counter()
    d, v = od.build_depth_map(np.stack([f.targets for f in fl]), np.stack([f.confidence for f in fl]), None,
                              e.pose.R, e.pose.center(), irow(e), np.stack([c.pose.R for c in cv]),
                              np.stack([c.pose.center() for c in cv]), [irow(c) for c in cv],
                              math.radians(2.0), 4, 0.05, 20, 1e-8)
    om.quantize(d, v)
    return d.size, time.perf_counter() - t0


def _cpu_lift_worker(job):
    """Oracle port of localize() for one generator-B query (lift + ransac)."""
    qi, wl, seed0 = job
    from oracle import lift as ol
    from oracle.geometry import q2R
    from oracle.posest import Config, ransac
    from synth_inputs import lifted_scene
    vmap, jobs, dc = lifted_scene(wl["K"], wl["queries"], wl["g"], seed=seed0, depth_kind=wl["depth"], only=[qi],
                                  fields="f32")
    t0 = time.perf_counter()
    pxs, Xs, ws = [], [], []
    for e in sorted(vmap.entries, key=lambda e: e.id):
        fp = jobs[0].fields[e.id]
        if dc is not None:
            vals, valid = dc[e.id].values.astype(np.float32), dc[e.id].valid
        else:
            q = e.qdepth
            vals, valid = ol.dequantize(q.codes, q.d_min, q.d_max, q.levels)
        f1 = (fp.db_to_query.targets, fp.db_to_query.confidence, fp.db_to_query.scale_x, fp.db_to_query.scale_y)
        f2 = (fp.query_to_db.targets, fp.query_to_db.confidence, fp.query_to_db.scale_x, fp.query_to_db.scale_y)
        I = e.intrinsics
        px, X, w = ol.lift(f1, f2, vals, valid, (I.fx, I.fy, I.cx, I.cy), (I.width, I.height),
                           q2R(e.pose.q), e.pose.t, 0.05)
        pxs.append(px)
        Xs.append(X)
        ws.append(w)
    I = jobs[0].intrinsics
    r = ransac(np.concatenate(pxs), np.concatenate(Xs), np.concatenate(ws), (I.fx, I.fy, I.cx, I.cy),
               Config(seed=query_seed(qi, seed0), max_iterations=wl["max_iterations"], miss_probability=wl["eta"]))
    return r.evals, time.perf_counter() - t0


def query_a(qi: int, n: int, outlier: float, sigma: float, seed0: int):
    """Deterministic generator-A query (test_posest.py:22-35 model, per-query GT pose)."""
    from synth_inputs import matches_a, random_pose
    rng = np.random.default_rng(seed0 + qi)
    _, R, t = random_pose(rng, 0.2, 0.2)
    px, X, w, _ = matches_a(n, outlier, sigma, seed=seed0 + 7919 * qi + 1, R=R, t=t)
    return px, X, w


def query_seed(qi: int, seed0: int) -> int:
    return 1_000_003 * seed0 + qi


# ----------------------------------------------------------------------------- CPU arm
def _cpu_worker(job):
    qi, wl, seed0 = job
    from oracle.posest import Config, ransac
    px, X, w = query_a(qi, wl["n"], wl["outlier"], wl["sigma"], seed0)
    t0 = time.perf_counter()
    r = ransac(px, X, w, (700.0, 700.0, 350.0, 350.0),
               Config(seed=query_seed(qi, seed0), max_iterations=wl.get("cpu_max_iterations", wl["max_iterations"]),
                      miss_probability=wl["eta"]))
    return r.evals, time.perf_counter() - t0


def cpu_sample(wl, seed0, n_queries, cores):
    """Run the oracle port on `n_queries` queries over `cores` processes; (evals, wall s)."""
    import multiprocessing as mp
    saved = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in saved:
        os.environ[k] = "1"
    lifted = "K" in wl
    worker = _cpu_map_worker if "E" in wl else (_cpu_lift_worker if lifted else _cpu_worker)
    n_queries = max(1, int(n_queries))
    cores = min(cores, n_queries)
    try:
        ctx = mp.get_context("spawn")
        with ctx.Pool(cores) as pool:
            if not lifted and "E" not in wl:
                pool.map(_cpu_worker, [(0, dict(wl, n=64, max_iterations=wl.get("batch", 1000),
                                                cpu_max_iterations=1000), seed0)] * cores)
            t0 = time.perf_counter()
            res = pool.map(worker, [(qi, wl, seed0) for qi in range(n_queries)])
            wall = time.perf_counter() - t0
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    # busy time per process (excludes input generation inside the workers)
    busy = sum(r[1] for r in res) / cores
    return sum(r[0] for r in res), min(wall, busy) if busy > 0 else wall


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_sample_plan(wl, cores):
    """(queries per sample, description) of the bounded CPU sample of a workload."""
    nq = max(1, int(round(cores * wl["cpu_queries_per_core"])))
    total = wl.get("queries", 1)
    parts = [f"{nq} quer{'y' if nq == 1 else 'ies'} of the workload (the first {nq}, same inputs and seeds)"]
    if wl.get("cpu_max_iterations"):
        parts.append(f"each truncated to its first {wl['cpu_max_iterations']} of {wl['max_iterations']} minimal "
                     f"samples (1/{wl['max_iterations'] // wl['cpu_max_iterations']} scale)")
    parts.append(f"{min(cores, nq)} processes (1 per core, BLAS 1 thread), oracle port")
    return nq, ", ".join(parts), nq < total or bool(wl.get("cpu_max_iterations"))


def cpu_baseline_line(wl, seed0, cores, evals=None, wall=None):
    """The ``cpu_baseline`` object: rate of the bounded sample, labelled."""
    nq, desc, extrapolated = cpu_sample_plan(wl, cores)
    if evals is None:
        evals, wall = cpu_sample(wl, seed0, nq, cores)
    out = {"value": evals / wall, "unit": "evals/s", "cores": min(cores, nq), "kind": "port",
           "sample": desc, "cpu_model": cpu_model(), "host_cores": cores,
           "sample_wall_s": wall, "queries_per_s": nq / wall}
    if extrapolated:
        out["extrapolated"] = True
        out["extrapolation"] = ("rate of the sample applied to the whole workload (queries are independent; "
                                "the metric is a rate)")
    return out


def run_reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = host_cores()
    if "E" in wl:
        run_map_reference_arm(args, wl, cores)
        return
    nq, desc, _ = cpu_sample_plan(wl, cores)
    seed0 = LIFT_SEED if "K" in wl else 3000
    # warm-up: the worker pool and imports on a small sample (one query per core)
    for _ in range(args.warmup):
        cpu_sample(dict(wl, cpu_max_iterations=wl.get("batch", 1000)) if "K" not in wl else wl, seed0,
                   min(nq, cores), cores)
    walls = []
    total_evals = 0
    for _ in range(args.steps):
        ev, wall = cpu_sample(wl, seed0, nq, cores)
        walls.append(wall)
        total_evals += ev
    value = total_evals / sum(walls)
    cpu = cpu_baseline_line(wl, seed0, cores, total_evals, sum(walls))
    line = {
        "impl": "reference", "metric": "hyp×corr evals/s", "value": value, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * statistics.mean(walls), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
        "config": {"workload": wl["name"], "queries_per_step": nq, "corrs_per_query": wl.get("n", "lifted")},
        "queries_per_s": nq / statistics.mean(walls),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_map_reference_arm(args, wl, cores):
    nm = min(wl["E"], max(1, int(cores * wl["cpu_maps_per_core"])))
    for _ in range(args.warmup):
        cpu_sample(wl, MAP_SEED, nm, cores)
    px = walls = 0.0
    ws = []
    for _ in range(args.steps):
        n, wall = cpu_sample(wl, MAP_SEED, nm, cores)
        px += n
        walls += wall
        ws.append(wall)
    value = px / walls
    line = {
        "impl": "reference", "metric": "depth-map px/s", "value": value, "unit": "px/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(ws),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["name"], "maps_per_step": nm},
        "cpu_baseline": {"value": value, "unit": "px/s", "cores": min(cores, nm), "kind": "port",
                         "sample": f"{nm} maps of the workload per step (1/core), oracle port",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "px/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
                pw.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w_max": max(pw) if pw else None, "samples": len(sm)}


# ----------------------------------------------------------------------------- timed regions
def timed_region(ctx, stream, sync_all, step, steps, profile):
    """Time `steps` calls of `step` with CUDA events on `stream` (barrier + sync
    on both sides).  profile=False is the reported measurement; profile=True
    repeats it with the library's per-stage CUDA events (stage breakdown and the
    scoring kernel's live launch time for the roofline).  Returns (ms,
    launches, stage profile or None, clocks)."""
    import torch
    ctx.profile(bool(profile))
    l0 = ctx.launches()
    sync_all()
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        sync_all()
    launches = ctx.launches() - l0
    prof = ctx.profile_read() if profile else None
    ctx.profile(False)
    return e0.elapsed_time(e1), launches, prof, clk.summary()


# ----------------------------------------------------------------------------- GPU arm: lifted
def serving_batch_ends(Q):
    """Micro-batch ends of the C5 serving loop (env VISLOC_C5_SIZES="a,b,..." overrides)."""
    env = os.environ.get("VISLOC_C5_SIZES")
    if env:
        return sorted({min(int(c), Q) for c in np.cumsum([int(x) for x in env.split(",")])} | {Q})
    from paper_2601_04185_b200.localizer import serving_schedule
    return serving_schedule(Q)


def run_lift_bench(args, wl, rank, world, local, dist):
    """C2 / C5: a step = lift (gate + depth decode + unproject) + batched LO-RANSAC
    for every query of the shard, device-resident fields/depth (value) or the
    full host API incl. field/depth H2D and result D2H (e2e)."""
    import torch
    from paper_2601_04185_b200 import _lib
    from paper_2601_04185_b200.localizer import LiftPlan
    from paper_2601_04185_b200.posest import RansacConfig
    from synth_inputs import lifted_scene

    from paper_2601_04185_b200.localizer import FieldPair, QueryJob
    from paper_2601_04185_b200.matchio import FieldArena, field_bytes

    Q = wl["queries"]
    seed0 = LIFT_SEED + 1000 * rank
    vmap, jobs, dcache = lifted_scene(wl["K"], Q, wl["g"], seed=seed0, depth_kind=wl["depth"], fields="f32")
    # the queries' fields arrive as IMLC payloads (matchio.py:9-20), one pinned
    # arena per micro-batch of queries (localizer.serving_schedule sizes); the GPU
    # lift reads the 12-B records in place
    from paper_2601_04185_b200.localizer import localize_pipelined
    ends = serving_batch_ends(Q)
    batches, q0 = [], 0
    bjobs = []
    for q1 in ends:
        order = [(qi, eid) for qi in range(q0, q1) for eid in sorted(jobs[qi].fields)]
        blobs = []
        for qi, eid in order:
            fp = jobs[qi].fields[eid]
            blobs += [field_bytes(fp.query_to_db), field_bytes(fp.db_to_query)]
        arena = FieldArena(blobs)
        del blobs
        bfields = {qi: {} for qi in range(q0, q1)}
        for k, (qi, eid) in enumerate(order):
            bfields[qi][eid] = FieldPair(arena[2 * k], arena[2 * k + 1])
        bj = [QueryJob(jobs[qi].query_id, jobs[qi].intrinsics, jobs[qi].descriptor, bfields[qi], jobs[qi].k_loc)
              for qi in range(q0, q1)]
        batches.append((bj, arena))
        bjobs += bj
        q0 = q1
    jobs = bjobs
    arena_bytes = sum(int(a.nbytes) for _, a in batches)
    seeds = [query_seed(qi, seed0) for qi in range(Q)]
    cfg = RansacConfig(max_iterations=wl["max_iterations"], miss_probability=wl["eta"])
    ctx = _lib.context(local)
    ctx.set_pruning(bool(wl.get("prune", True)))  # (the context outlives the previous config's setting)
    stream = torch.cuda.current_stream()
    for _, a in batches:
        a.device()  # device-resident copies for the `value` path
    dev_cache = {}  # the map's depth stays resident in HBM across steps (server state)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    plan = LiftPlan(jobs, vmap, depth_cache=dcache, device_cache=dev_cache)
    out = None
    for _ in range(args.warmup):
        out, run, offsets, _ = plan.run_device(cfg, seeds, out=None)
    stats = out["stats"].cpu().numpy()
    evals_per_step = int(stats[:, 2].sum())
    matches = int(offsets[-1])
    conv_rate = float(out["converged"].float().mean().item())
    def step():
        plan.run_device(cfg, seeds)

    ms, launches, _, clocks = timed_region(ctx, stream, sync_all, step, args.steps, False)
    ctx.scoring_counters(reset=True)
    ms_prof, _, prof, _ = timed_region(ctx, stream, sync_all, step, args.steps, True)
    skipped, tail_evals = ctx.scoring_counters(reset=True)
    executed_per_step = evals_per_step - skipped / args.steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    ev = torch.tensor([float(evals_per_step)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ev)
    ms_max = float(t.item())
    value = float(ev.item()) * args.steps / (ms_max / 1e3)
    qps = Q * world * args.steps / (ms_max / 1e3)

    e2e = None
    if not args.no_e2e:
        big = max(a.host.numel() for _, a in batches)
        lanes = int(os.environ.get("VISLOC_PIPE_LANES", 2))
        bufs = [torch.empty(big, dtype=torch.uint8, device="cuda") for _ in range(int(os.environ.get("VISLOC_PIPE_BUFS", lanes + 1)))]

        def e2e_step():
            # micro-batched serving loop: batch k+1's IMLC payloads (pinned) go
            # to HBM on a copy stream while batch k is retrieved, lifted and
            # estimated; results come back to the host per batch
            return localize_pipelined(batches, vmap, cfg, seeds=seeds, depth_cache=dcache, device_cache=dev_cache,
                                      retrieval="gpu", buffers=bufs)

        for _ in range(2):  # warm the pinned result pool the loop cycles through
            res = e2e_step()
        sync_all()
        e0.record(stream)
        for _ in range(args.steps):
            res = None  # the caller is done with the previous step's results
            res = e2e_step()
        e1.record(stream)
        sync_all()
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        h2d = arena_bytes
        d2h = sum(int(r.inlier_flags.size) + 7 * 8 + 5 * 8 for r in res)
        e2e = {"value": float(ev.item()) * args.steps / (float(et.item()) / 1e3), "unit": "evals/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "queries_per_s": Q * world * args.steps / (float(et.item()) / 1e3)}

    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    props = torch.cuda.get_device_properties(local)
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = props.multi_processor_count * 128 * 2 * sm_max * 1e6 / 1e12
    score_ms, score_launches = prof["score"]
    lift_ms, lift_launches = prof["lift"]
    # executed evaluations (exact pruning skips some) over the scoring stage's time
    achieved = (executed_per_step * args.steps * FLOP_PER_EVAL) / (score_ms / 1e3) / 1e12 if score_ms else None
    ms = ms_prof  # shares below are of the profiled region
    # lift algorithmic bytes per step: IMLC record 12 B/cell (f32 fields), depth taps, 48 B per match out
    # (px 2 f64, X 3 f64, w f64 — the rows the estimator reads; no per-match entry ids are written)
    tap_bytes = {"f32": 5, "f16": 3, "u8": 1}[wl["depth"]]
    lift_bytes = 12 * plan.cells + matches * (48 + 2.5 * tap_bytes)
    hbm = float(peaks.get("hbm_gbs", 6548.8))
    lift_gbs = lift_bytes * args.steps / (lift_ms / 1e3) / 1e9 if lift_ms else None
    roof = {"bound": "fp32", "kernel": "k_score", "achieved": achieved, "peak": round(fp32_peak, 2),
            "unit": "TFLOP/s", "frac": (achieved / fp32_peak) if achieved else None,
            "peak_source": "derived SMs*128*2*sm_max_mhz (MEASURED_PEAKS.json has no FP32 entry)",
            "traffic": None, "score_share_of_step": score_ms / ms if ms else None,
            "evals_nominal_per_step": evals_per_step, "evals_executed_per_step": executed_per_step,
            "evals_tail_per_step": tail_evals / args.steps,
            "lift": {"bound": "hbm", "achieved": lift_gbs, "peak": hbm, "unit": "GB/s",
                     "frac": (lift_gbs / hbm) if lift_gbs else None, "algorithmic_bytes_per_step": lift_bytes,
                     "share_of_step": lift_ms / ms if ms else None, "launches": lift_launches}}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_line(wl, seed0, host_cores())
        cpu["sample"] += " (lift + ransac per query)"
    if rank == 0:
        line = {
            "metric": "hyp×corr evals/s", "value": value, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64",
            "data": "synthetic",
            "config": {"workload": wl["name"], "queries_per_gpu": Q, "db_images": wl["K"], "grid": wl["g"],
                       "lifted_corrs_per_step": matches, "depth": wl["depth"],
                       "fields": f"IMLC f32 records, {arena_bytes / 1e9:.3f} GB/step in pinned arenas, "
                                 f"micro-batches {ends}",
                       "map": "depth resident in HBM (uploaded once); e2e H2D = the field payloads",
                       "scoring": "exact prefix pruning (product default; outputs identical to full scoring; value "
                                  "counts the reference's nominal evaluations, the roofline the executed ones)",
                       "l2": f"fields {plan.field_bytes / 1e9:.2f} GB/GPU",
                       "parallelism": f"query-sharded x{world}, no collective"},
            "queries_per_s": qps, "converged_frac": conv_rate, "e2e": e2e, "roofline": roof,
            "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": launches,
            "stage_ms_per_step": {k: round(v[0] / args.steps, 3) for k, v in prof.items()},
            "profiled_ms_per_step": ms_prof / args.steps,
        }
        return line
    return None


# ----------------------------------------------------------------------------- GPU arm: mapping
def run_map_bench(args, wl, rank, world, local, dist):
    """Mapping: a step = triangulate every entry's depth map (one vl_build_depth_maps
    launch) + quantise them all (one vl_quantize_depth launch), fields resident
    in HBM (value) or uploaded from pinned host memory with depth codes read
    back (e2e, build_map_from_fields's device work)."""
    import torch
    from paper_2601_04185_b200 import _lib
    from paper_2601_04185_b200.depthbuild import DepthBuildPlan, TriangulationConfig
    from paper_2601_04185_b200.mapstore import quantize_depth_device
    from synth_inputs import mapping_scene

    seed0 = MAP_SEED + 1000 * rank
    jobs = mapping_scene(wl["E"], wl["V"], wl["g"], seed=seed0)
    cfg = TriangulationConfig()
    ctx = _lib.context(local)
    stream = torch.cuda.current_stream()

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    plan = DepthBuildPlan(jobs, cfg)
    for _ in range(args.warmup):
        codes = quantize_depth_device(plan.run().device_maps())
    valid_frac = float(plan.valid.float().mean().item())

    def step():
        quantize_depth_device(plan.run().device_maps())

    ms, launches, _, clocks = timed_region(ctx, stream, sync_all, step, args.steps, False)
    # kernel-only time of the triangulation launch (live CUDA events on the launching stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sync_all()
    e0.record(stream)
    for _ in range(args.steps):
        plan.run()
    e1.record(stream)
    sync_all()
    tri_ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    px = plan.pixels
    value = px * world * args.steps / (ms_max / 1e3)

    e2e = None
    if not args.no_e2e:
        def e2e_step():
            p = DepthBuildPlan(jobs, cfg).run()
            cs = quantize_depth_device(p.device_maps())
            return [c.cpu() for c in cs], p.field_bytes
        e2e_step()
        sync_all()
        e0.record(stream)
        for _ in range(args.steps):
            out, h2d = e2e_step()
        e1.record(stream)
        sync_all()
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": px * world * args.steps / (float(et.item()) / 1e3), "unit": "px/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(sum(c.numel() for c in out))}
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    props = torch.cuda.get_device_properties(local)
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp64_peak = props.multi_processor_count * 64 * 2 * sm_max * 1e6 / 1e12
    votes = px * wl["V"] * wl["V"]
    achieved = votes * VOTE_FLOP / (tri_ms / 1e3) / 1e12
    roof = {"bound": "fp64", "kernel": "k_tri_map", "achieved": achieved, "peak": round(fp64_peak, 2),
            "unit": "TFLOP/s", "frac": achieved / fp64_peak,
            "peak_source": "derived SMs*64*2*sm_max_mhz (MEASURED_PEAKS.json has no FP64 entry)",
            "flop_per_vote": VOTE_FLOP, "votes_per_s": votes / (tri_ms / 1e3),
            "note": "vote-stage FLOPs only (the Newton refinement, most of the work, is excluded from the "
                    "count); ncu_fp64_pipe_active is the measured FP64-pipe utilisation of the whole kernel",
            "ncu_fp64_pipe_active": 0.234, "ncu_source": "profiles/r01c_k_tri_quant_full_raw.csv "
            "(sm__pipe_fp64_cycles_active, ncu --set full of bench.py --workload map)",
            "traffic": None, "tri_ms_per_step": tri_ms, "share_of_step": tri_ms / (ms / args.steps)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = host_cores()
        nm = min(wl["E"], cores * wl["cpu_maps_per_core"])
        n, wall = cpu_sample(wl, MAP_SEED, nm, cores)
        cpu = {"value": n / wall, "unit": "px/s", "cores": min(cores, nm), "kind": "port",
               "sample": f"{nm} maps of the same workload (oracle build_depth_map + quantize), 1 process/map"}
    if rank == 0:
        print(json.dumps({
            "metric": "depth-map px/s", "value": value, "unit": "px/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["name"], "maps_per_gpu": wl["E"], "views": wl["V"], "grid": wl["g"],
                       "pixels_per_step": px, "valid_frac": valid_frac,
                       "l2": f"fields {plan.field_bytes / 1e6:.0f} MB/GPU resident",
                       "parallelism": f"map-sharded x{world}, no collective"},
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": launches,
        }), flush=True)


# ----------------------------------------------------------------------------- GPU arm: generator A
def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def bench_direct(args, wl, rank, world, local, dist, steps, mode="weak", with_e2e=True, with_cpu=True):
    """Generator-A workloads (C1, C3, C3a, C4).  mode "weak": every rank runs
    its own wl["queries"] queries; "strong": the wl["queries"] queries of the
    job are split across the ranks (interleaved, dist.shard_indices).
    Returns the JSON line (rank 0) or None."""
    import torch

    from paper_2601_04185_b200 import _lib
    from paper_2601_04185_b200.dist import shard_indices
    from paper_2601_04185_b200.geometry import CameraIntrinsics
    from paper_2601_04185_b200.posest import (RansacConfig, ransac_pnp, ransac_pnp_device, ransac_pnp_host,
                                              ransac_pnp_stream)
    n = wl["n"]
    if mode == "strong":
        seed0 = 3000
        qids = shard_indices(wl["queries"], rank, world, "interleaved")
    else:
        seed0 = 3000 + 100_000 * rank
        qids = list(range(wl["queries"]))
    Q = len(qids)
    qs = [query_a(qi, n, wl["outlier"], wl["sigma"], seed0) for qi in qids]
    px_h = torch.from_numpy(np.concatenate([q[0] for q in qs])).pin_memory()
    X_h = torch.from_numpy(np.concatenate([q[1] for q in qs])).pin_memory()
    w_h = torch.from_numpy(np.concatenate([q[2] for q in qs])).pin_memory()
    single = [(q[0], q[1], q[2]) for q in qs] if Q == 1 else None
    del qs
    offsets = np.arange(Q + 1, dtype=np.int64) * n
    intr1 = CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
    intr = [intr1] * Q
    seeds = [query_seed(qi, seed0) for qi in qids]
    cfg = RansacConfig(max_iterations=wl["max_iterations"], miss_probability=wl["eta"])
    px_d, X_d, w_d = px_h.cuda(), X_h.cuda(), w_h.cuda()
    ctx = _lib.context(local)
    prune = bool(wl.get("prune", True))
    ctx.set_pruning(prune)
    stream = torch.cuda.current_stream()

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(v, op="max"):
        t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    out = None
    for _ in range(args.warmup):
        out = ransac_pnp_device(px_d, X_d, w_d, offsets, intr, seeds, cfg, out=out)
    stats0 = out["stats"].cpu().numpy()
    evals_per_step = int(stats0[:, 2].sum())
    conv_rate = float(out["converged"].float().mean().item())

    # ---- device-resident timed region (value), then the same steps profiled
    def step():
        ransac_pnp_device(px_d, X_d, w_d, offsets, intr, seeds, cfg, out=out)

    ms, launches, _, clocks = timed_region(ctx, stream, sync_all, step, steps, False)
    ctx.scoring_counters(reset=True)
    ms_prof, _, prof, _ = timed_region(ctx, stream, sync_all, step, steps, True)
    skipped, tail_evals = ctx.scoring_counters(reset=True)
    executed_per_step = evals_per_step - skipped / steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms_max = max_over_ranks(ms)
    evals_total = max_over_ranks(evals_per_step, "sum") * steps
    q_total = max_over_ranks(Q, "sum")
    value = evals_total / (ms_max / 1000.0)
    queries_per_s = q_total * steps / (ms_max / 1000.0)

    # ---- end-to-end through the public host API
    e2e = None
    if with_e2e and Q == 1:
        # the drop-in call a user makes: ransac_pnp(matches (host numpy), intr, cfg) -> PoseEstimate
        px1, X1, w1 = single[0]
        c1 = RansacConfig(max_iterations=wl["max_iterations"], miss_probability=wl["eta"], seed=seeds[0])
        for _ in range(2):
            est = ransac_pnp((px1, X1, w1), intr1, c1)
        sync_all()
        e0.record(stream)
        for _ in range(steps):
            est = ransac_pnp((px1, X1, w1), intr1, c1)
        e1.record(stream)
        sync_all()
        ems = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": evals_total / (ems / 1000.0), "unit": "evals/s",
               "h2d_bytes_per_step": int(px1.nbytes + X1.nbytes + w1.nbytes),
               "d2h_bytes_per_step": int(est.inlier_flags.size + 8 * (4 + 3 + 1 + 1 + 1 + 1 + 4)),
               "api": "ransac_pnp((px, X, w) host numpy, intr, cfg) -> PoseEstimate (the drop-in call), "
                      "per call: pinned staging, H2D, estimate, D2H",
               "latency_ms": ems / steps, "queries_per_s": q_total * steps / (ems / 1000.0)}
    elif with_e2e:
        # one-shot: one ransac_pnp_host call (the whole batch's H2D, staged
        # admission, estimate, D2H of every result), nothing overlapped from
        # before; a first call warms the device / pinned allocations
        host, hb, db = ransac_pnp_host(px_h, X_h, w_h, offsets, intr, seeds, cfg)
        del host
        sync_all()
        t0 = time.perf_counter()
        e0.record(stream)
        host, hb, db = ransac_pnp_host(px_h, X_h, w_h, offsets, intr, seeds, cfg)
        e1.record(stream)
        sync_all()
        one_ms = max_over_ranks(max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)))
        one_shot = {"value": evals_total / steps / (one_ms / 1000.0), "unit": "evals/s", "ms": one_ms,
                    "h2d_bytes": int(hb), "d2h_bytes": int(db),
                    "api": "ransac_pnp_host: one call after a warm-up call, the batch's whole H2D inside (nothing "
                           "overlapped from a previous batch: the pipeline fill is included)"}
        del host
        # serving loop: every step is one batch of Q queries copied from pinned
        # host memory (H2D) and its results read back (D2H); batch k+1's copy
        # streams while batch k is estimated
        batch = (px_h, X_h, w_h, offsets, intr, seeds)
        for res in ransac_pnp_stream([batch] * 3, cfg):  # warm (device buffers, pinned result sets)
            del res
        sync_all()
        W = 3
        h2d = d2h = 0
        gen = ransac_pnp_stream([batch] * (W + steps + 1), cfg)
        for i, (res, hb, db) in enumerate(gen):
            h2d, d2h = hb, db
            del res  # results consumed: the pinned set goes back to the pool
            if i == W - 1:
                e0.record(stream)
            if i == W - 1 + steps:
                e1.record(stream)
                break
        gen.close()
        sync_all()
        ems = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": evals_total / (ems / 1000.0), "unit": "evals/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "api": "ransac_pnp_stream: one batch per step, batch k+1 H2D overlaps batch k; steady state "
                      "(timed from the 3rd result handed out, pipeline fill and drain excluded; see one_shot)",
               "queries_per_s": q_total * steps / (ems / 1000.0), "one_shot": one_shot}

    # ---- roofline of the dominant kernel (fp32 MSAC scoring), live CUDA events
    peaks = _peaks()
    props = torch.cuda.get_device_properties(local)
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = props.multi_processor_count * 128 * 2 * sm_max * 1e6 / 1e12
    score_ms, score_launches = prof["score"]
    # executed evaluations (= nominal unless pruning skipped some) over the scoring stage's time
    achieved = (executed_per_step * steps * FLOP_PER_EVAL) / (score_ms / 1000.0) / 1e12 if score_ms else None
    stage_ms = {k: round(v[0] / steps, 3) for k, v in prof.items()}
    traffic = None
    try:  # DRAM bytes per k_score launch from the committed ncu --set full capture (profiles/)
        tr = json.loads((ROOT / "profiles" / "traffic.json").read_text())["k_score"]
        if tr.get("workload") == args.workload and Q == 1000 and mode == "weak":
            traffic = {"dram_bytes_per_launch": tr["dram_bytes_per_launch"], "source": tr["source"],
                       "algorithmic_bytes_per_launch": int(evals_per_step / score_launches * steps
                                                           / 10_000 * (48 + 4 * 20)) +
                       (Q * 10_000 * 24 if score_launches else 0)}  # 24-B records (pair-packed f32)
    except Exception:
        traffic = None
    roof = {"bound": "fp32", "kernel": "k_score", "achieved": achieved, "peak": round(fp32_peak, 2),
            "unit": "TFLOP/s", "frac": (achieved / fp32_peak) if achieved else None,
            "peak_source": "derived SMs*128*2*sm_max_mhz (MEASURED_PEAKS.json has no FP32 entry)",
            "flop_per_eval": FLOP_PER_EVAL,
            "traffic": traffic["dram_bytes_per_launch"] if traffic else None, "traffic_detail": traffic,
            "evals_per_s_kernel": (executed_per_step * steps) / (score_ms / 1000.0) if score_ms else None,
            "score_share_of_step": (score_ms / ms_prof) if ms_prof else None,
            "score_launches": score_launches,
            "evals_nominal_per_step": evals_per_step, "evals_executed_per_step": executed_per_step,
            "evals_tail_per_step": tail_evals / steps}
    if prune and skipped:
        roof["kernel"] = "k_score + k_score_tail (pruned rounds)"

    cpu = None
    if rank == 0 and world == 1 and with_cpu and not args.no_cpu:
        cpu = cpu_baseline_line(wl, seed0, host_cores())
    if rank != 0:
        return None
    return {
        "metric": "hyp×corr evals/s", "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms_max / steps,
        "higher_is_better": True, "scaling": mode, "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic",
        "config": {"workload": wl["name"], "queries_total": int(q_total),
                   "queries_per_gpu": Q if mode == "weak" else f"{wl['queries']}/{world} (interleaved)",
                   "corrs_per_query": n, "n_sub": min(n, 10_000), "max_iterations": wl["max_iterations"],
                   "miss_probability": wl["eta"],
                   "scoring": ("exact prefix pruning (vl_set_scoring_pruning; outputs identical to full scoring; "
                               "value counts the reference's nominal hyp x corr evaluations, the roofline the "
                               "executed ones)" if prune else
                               "full: every hypothesis scored on the whole subset, as the reference does"),
                   "l2": (f"inputs {px_h.numel() * 8 * 3 / 1e9:.2f} GB/GPU (> 126 MB L2; no flush needed)"
                          if px_h.numel() * 24 > 126e6 else
                          f"inputs {px_h.numel() * 24 / 1e6:.2f} MB/GPU, L2-resident (single-query latency "
                          f"config: every step re-reads them from L2, as a serving loop would)"),
                   "parallelism": f"query-sharded x{world} ({'weak' if mode == 'weak' else 'strong, interleaved'}), "
                                  f"no collective"},
        "queries_per_s": queries_per_s, "converged_frac": conv_rate,
        "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
        "clocks": clocks, "gpu_launches": launches, "stage_ms_per_step": stage_ms,
        "profiled_ms_per_step": ms_prof / steps,
    }


def _config_summary(line):
    """The parts of a workload's line that the default line's ``configs`` carries."""
    keep = ("value", "unit", "ms_per_step", "steps", "queries_per_s", "converged_frac", "e2e", "roofline",
            "cpu_baseline", "clocks", "gpu_launches", "stage_ms_per_step", "config")
    return {k: line[k] for k in keep if k in line}


# ----------------------------------------------------------------------------- launcher
def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n: int) -> int:
    """Re-launch this command under torch.distributed.run with n ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(args):
    """(rank, world, local device, backend) from the torchrun environment; initialises the group."""
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # VISLOC_BENCH_BACKEND=gloo: functional check of the multi-rank path on
    # fewer GPUs than ranks (ranks share devices: never a measurement)
    backend = os.environ.get("VISLOC_BENCH_BACKEND", "nccl")
    dry = bool(os.environ.get("VISLOC_BENCH_DRYRUN"))
    if not dry:
        ndev = torch.cuda.device_count()
        if ndev == 0:
            raise SystemExit("bench.py: no CUDA device (the GPU arm has no CPU fallback)")
        if "VISLOC_BENCH_DEVICE" in os.environ:
            local = int(os.environ["VISLOC_BENCH_DEVICE"])
        elif backend != "nccl":
            local %= ndev
        elif local >= ndev:
            raise SystemExit(f"bench.py: rank {rank} needs GPU {local} but only {ndev} are visible "
                             f"(use VISLOC_BENCH_BACKEND=gloo for a functional check)")
        torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl" and not dry:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo" if dry else backend)
    return rank, world, local, backend, dist


def dry_run(args, rank, world, dist):
    """CPU check of the launcher: N ranks come up, own interleaved shards that
    partition the job, and reduce a time as a max over ranks."""
    import torch

    from paper_2601_04185_b200.dist import shard_indices
    mine = shard_indices(1000, rank, world, "interleaved")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    cnt = torch.tensor([float(len(mine))], dtype=torch.float64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(cnt)
    if rank == 0:
        print(json.dumps({"dryrun": True, "n_gpus": world, "max_over_ranks": float(t.item()),
                          "queries_total": int(cnt.item()), "world_env": os.environ.get("WORLD_SIZE")}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + sorted(LIFT_WORKLOADS) + sorted(MAP_WORKLOADS),
                    default="c3")
    ap.add_argument("--queries", type=int, default=None, help="override queries per GPU")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="default line without the C1/C4/C5 configs")
    args = ap.parse_args()
    lifted = args.workload in LIFT_WORKLOADS
    mapping = args.workload in MAP_WORKLOADS
    wl = dict(MAP_WORKLOADS[args.workload] if mapping else
              LIFT_WORKLOADS[args.workload] if lifted else WORKLOADS[args.workload])
    if args.queries:
        wl["queries"] = args.queries
    if args.impl == "reference":
        run_reference_arm(args, wl)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)

    rank, world, local, backend, dist = dist_setup(args)
    if os.environ.get("VISLOC_BENCH_DRYRUN"):
        dry_run(args, rank, world, dist)
        if world > 1:
            dist.destroy_process_group()
        return 0
    if lifted or mapping:
        if mapping:
            run_map_bench(args, wl, rank, world, local, dist)
        else:
            line = run_lift_bench(args, wl, rank, world, local, dist)
            if line is not None:
                print(json.dumps(line), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return 0

    line = bench_direct(args, wl, rank, world, local, dist, args.steps, "weak", not args.no_e2e)
    if world > 1 and args.workload in ("c3", "c3a"):
        # the literal BASELINE C3 batch (1000 queries) split across the ranks
        strong = bench_direct(args, wl, rank, world, local, dist, args.steps, "strong", False, False)
        if rank == 0:
            line["strong"] = {k: strong[k] for k in ("value", "unit", "ms_per_step", "queries_per_s", "config",
                                                     "roofline", "clocks")}
    if world == 1 and args.workload == "c3" and not args.no_configs:
        # the other BASELINE configs, each with its own value / e2e / roofline / cpu_baseline
        configs = {}
        sub = bench_direct(args, dict(WORKLOADS["c3p"]), rank, world, local, dist, args.steps, "weak",
                           not args.no_e2e, False)
        configs["c3p"] = _config_summary(sub)
        for name in ("c3a", "c1", "c4"):
            sub = bench_direct(args, dict(WORKLOADS[name]), rank, world, local, dist, args.steps, "weak",
                               not args.no_e2e)
            configs[name] = _config_summary(sub)
        sub = run_lift_bench(argparse.Namespace(**{**vars(args), "workload": "c5"}), dict(LIFT_WORKLOADS["c5"]),
                             rank, world, local, dist)
        configs["c5"] = _config_summary(sub)
        line["configs"] = configs
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
