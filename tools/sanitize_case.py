"""Small end-to-end cases for compute-sanitizer runs (tools only).

1 and 3 queries (clustered launches, the pipelined round loop on two
streams) and a 24-query batch of 12k correspondences (coarse scoring
items: exact pruning with the split first round, k_score_tail).
"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402
import paper_2601_04185_b200 as vl  # noqa: E402
from synth_inputs import batch_a  # noqa: E402

intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
pxs, Xs, ws = batch_a(3, 600, 0.5, 1.0, seed0=5)
cfg = vl.RansacConfig(max_iterations=2000, miss_probability=1e-300)
r1 = vl.ransac_pnp((pxs[0], Xs[0], ws[0]), intr, cfg)
r3 = vl.ransac_pnp_batch(list(zip(pxs, Xs, ws)), intr, cfg, seeds=[1, 2, 3])
pxb, Xb, wb = batch_a(24, 12_000, 0.7, 1.0, seed0=9)
rb = vl.ransac_pnp_batch(list(zip(pxb, Xb, wb)), intr, vl.RansacConfig(max_iterations=3000, miss_probability=1e-300),
                         seeds=list(range(24)))
print("ok", r1.converged, [r.converged for r in r3], sum(r.converged for r in rb))
