"""Wall-clock phase breakdown of the C5 end-to-end path (localize_batch over IMLC arenas).

GPU only:  python tools/lift_pipe.py [c5|c2]
"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import bench  # noqa: E402
from paper_2601_04185_b200 import localizer as L  # noqa: E402
from paper_2601_04185_b200.matchio import FieldArena, field_bytes  # noqa: E402
from paper_2601_04185_b200.posest import RansacConfig, _estimates_from  # noqa: E402
from synth_inputs import lifted_scene  # noqa: E402


def main():
    wl = bench.LIFT_WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
    Q = wl["queries"]
    vmap, jobs, dcache = lifted_scene(wl["K"], Q, wl["g"], seed=bench.LIFT_SEED, depth_kind=wl["depth"],
                                      fields="f32")
    order = [(qi, eid) for qi, job in enumerate(jobs) for eid in sorted(job.fields)]
    blobs = []
    for qi, eid in order:
        fp = jobs[qi].fields[eid]
        blobs += [field_bytes(fp.query_to_db), field_bytes(fp.db_to_query)]
    arena = FieldArena(blobs)
    bf = [dict() for _ in jobs]
    for k, (qi, eid) in enumerate(order):
        bf[qi][eid] = L.FieldPair(arena[2 * k], arena[2 * k + 1])
    jobs = [L.QueryJob(j.query_id, j.intrinsics, j.descriptor, f, j.k_loc) for j, f in zip(jobs, bf)]
    seeds = [bench.query_seed(qi, bench.LIFT_SEED) for qi in range(Q)]
    cfg = RansacConfig(max_iterations=wl["max_iterations"], miss_probability=wl["eta"])
    dev = torch.empty(arena.host.numel(), dtype=torch.uint8, device="cuda")
    cs = torch.cuda.Stream()
    dc = {}
    for rep in range(4):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        arena.upload(dev, stream=cs)
        t.append(time.perf_counter())
        plan = L.LiftPlan(jobs, vmap, None, dcache, dc, 0.05, "gpu")
        t.append(time.perf_counter())
        start, end = plan.lift()
        t.append(time.perf_counter())
        out, run, offsets, _ = plan.run_device(cfg, seeds)  # lifts again + estimates
        t.append(time.perf_counter())
        res = _estimates_from(out, offsets)
        t.append(time.perf_counter())
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        names = ["upload-issue", "plan", "lift(sync)", "lift+ransac", "estimates(D2H)", "tail"]
        print(rep, " ".join(f"{n}={1e3 * (b - a):.2f}" for n, a, b in zip(names, t, t[1:])),
              f"total={1e3 * (t[-1] - t[0]):.2f} ms", len(res))


if __name__ == "__main__":
    main()
