"""Wall-clock breakdown of the C5 serving step by host function (tools only).

Wraps the localizer's per-batch pieces with perf_counter accumulators (no
profiler overhead) and runs bench.py's C5 e2e step.  Blocking calls (lift
counts, the RANSAC round loop, result reads) absorb GPU time.  GPU only:
    python tools/c5_host_breakdown.py [workload] [steps]
"""
import sys
import time
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import bench  # noqa: E402

ACC = defaultdict(float)
CNT = defaultdict(int)
TL = []  # (label, host t, cuda event) timeline of one step
TRACE = [False]


def wrap(obj, name, label=None):
    fn = getattr(obj, name)
    label = label or name

    def w(*a, **k):
        t0 = time.perf_counter()
        if TRACE[0]:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            TL.append((label + " >", t0, ev))
        try:
            return fn(*a, **k)
        finally:
            t1 = time.perf_counter()
            ACC[label] += t1 - t0
            CNT[label] += 1
            if TRACE[0]:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                TL.append((label + " <", t1, ev))
    setattr(obj, name, w)


def main():
    wl = dict(bench.LIFT_WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c5"])
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    from paper_2601_04185_b200 import localizer as L
    from paper_2601_04185_b200 import posest as P
    from paper_2601_04185_b200.localizer import FieldPair, QueryJob, localize_pipelined
    from paper_2601_04185_b200.matchio import FieldArena, field_bytes
    from paper_2601_04185_b200.posest import RansacConfig, _stage_schedule
    from synth_inputs import lifted_scene
    Q = wl["queries"]
    vmap, jobs, dcache = lifted_scene(wl["K"], Q, wl["g"], seed=bench.LIFT_SEED, depth_kind=wl["depth"],
                                      fields="f32")
    ends = bench.serving_batch_ends(Q)
    batches, q0 = [], 0
    for q1 in ends:
        order = [(qi, eid) for qi in range(q0, q1) for eid in sorted(jobs[qi].fields)]
        blobs = []
        for qi, eid in order:
            fp = jobs[qi].fields[eid]
            blobs += [field_bytes(fp.query_to_db), field_bytes(fp.db_to_query)]
        arena = FieldArena(blobs)
        bf = {qi: {} for qi in range(q0, q1)}
        for k, (qi, eid) in enumerate(order):
            bf[qi][eid] = FieldPair(arena[2 * k], arena[2 * k + 1])
        batches.append(([QueryJob(jobs[qi].query_id, jobs[qi].intrinsics, jobs[qi].descriptor, bf[qi],
                                  jobs[qi].k_loc) for qi in range(q0, q1)], arena))
        q0 = q1
    cfg = RansacConfig(max_iterations=wl["max_iterations"], miss_probability=wl["eta"])
    seeds = [bench.query_seed(qi, bench.LIFT_SEED) for qi in range(Q)]
    dev_cache = {}
    big = max(a.host.numel() for _, a in batches)
    import os
    bufs = [torch.empty(big, dtype=torch.uint8, device="cuda")
            for _ in range(int(os.environ.get("VISLOC_PIPE_BUFS", int(os.environ.get("VISLOC_PIPE_LANES", 2)) + 1)))]

    def step():
        return localize_pipelined(batches, vmap, cfg, seeds=seeds, depth_cache=dcache, device_cache=dev_cache,
                                  retrieval="gpu", buffers=bufs)
    step()
    torch.cuda.synchronize()
    import gc
    import os
    if os.environ.get("GCMODE") == "freeze":
        gc.freeze()
    elif os.environ.get("GCMODE") == "off":
        gc.disable()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    base = (time.perf_counter() - t0) / steps * 1e3
    print(f"e2e step (unwrapped): {base:.2f} ms  batches/step {len(batches)}")
    for name in ("_retrieve", "_plan", "_seg_table", "_call_lift", "ransac_pnp_device", "_estimates_from",
                 "localize_batch", "_device_depth"):
        wrap(L, name)
    wrap(L._FieldUpload, "__init__", "_FieldUpload")
    wrap(L.LiftPlan, "__init__", "LiftPlan.__init__")
    wrap(L.LiftPlan, "lift", "LiftPlan.lift")
    wrap(L, "_stage_results")
    from paper_2601_04185_b200.matchio import FieldArena as FA
    orig_upload = FA.upload

    def upload(self, out, stream=None):
        if TRACE[0] and stream is not None:
            a = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            TL.append((f"upload {self.nbytes >> 20} MB >", time.perf_counter(), a))
        r = orig_upload(self, out, stream)
        if TRACE[0] and stream is not None:
            b = torch.cuda.Event(enable_timing=True)
            b.record(stream)
            TL.append((f"upload {self.nbytes >> 20} MB <", time.perf_counter(), b))
        return r
    FA.upload = upload
    wrap(L.LiftPlan, "collect", "collect")
    step()
    torch.cuda.synchronize()
    ACC.clear(); CNT.clear()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) / steps * 1e3
    print(f"e2e step (wrapped): {tot:.2f} ms")
    for k, v in sorted(ACC.items(), key=lambda kv: -kv[1]):
        print(f"  {k:24s} {v / steps * 1e3:8.3f} ms/step  ({CNT[k] // steps} calls/step)")
    # one traced step: host wall time vs GPU stream time of every wrapped call
    torch.cuda.synchronize()
    TRACE[0] = True
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    print("timeline (host ms | gpu-stream ms at the same point):")
    for label, t, ev in sorted(TL, key=lambda x: x[1]):
        print(f"  {(t - h0) * 1e3:8.3f} | {e0.elapsed_time(ev):8.3f}  {label}")


if __name__ == "__main__":
    main()
