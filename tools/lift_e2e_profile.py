"""Host-side profile of the C5 serving step (localize_pipelined) — tools only.

Runs bench.py's C5 setup, then cProfile over a few e2e steps; prints the top
functions by cumulative and own time.  GPU only:
    python tools/lift_e2e_profile.py [workload]
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import bench  # noqa: E402


def main():
    wl = dict(bench.LIFT_WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c5"])
    from paper_2601_04185_b200.localizer import FieldPair, QueryJob, localize_pipelined
    from paper_2601_04185_b200.matchio import FieldArena, field_bytes
    from paper_2601_04185_b200.posest import RansacConfig, _stage_schedule
    from synth_inputs import lifted_scene
    Q = wl["queries"]
    vmap, jobs, dcache = lifted_scene(wl["K"], Q, wl["g"], seed=bench.LIFT_SEED, depth_kind=wl["depth"],
                                      fields="f32")
    ends = _stage_schedule(Q)
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
    bufs = [torch.empty(big, dtype=torch.uint8, device="cuda") for _ in range(2)]

    def step():
        return localize_pipelined(batches, vmap, cfg, seeds=seeds, depth_cache=dcache, device_cache=dev_cache,
                                  retrieval="gpu", buffers=bufs)
    step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    print(f"e2e step: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(18)
    st.sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
