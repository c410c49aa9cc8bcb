"""k_final A/B: TMA-streamed full-set passes (VISLOC_FINAL_STAGED=1) vs plain loads, one-CTA-per-query batch."""
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402
import paper_2601_04185_b200 as vl  # noqa: E402
from synth_inputs import batch_a  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 160
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3001
intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
pxs, Xs, ws = batch_a(nq, n, 0.5, 1.0, seed0=5)
cfg = vl.RansacConfig(max_iterations=2000, miss_probability=1e-300)
res = {}
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["1"]
for st in ["0"] + modes:
    os.environ["VISLOC_FINAL_STAGED"] = st
    res[st] = vl.ransac_pnp_batch(list(zip(pxs, Xs, ws)), intr, cfg, seeds=list(range(nq)))
    print("staged", st, "done", flush=True)
for md in modes:
  bad = 0
  for a, b in zip(res["0"], res[md]):
    same = (np.array_equal(a.inlier_flags, b.inlier_flags) and a.inlier_count == b.inlier_count
            and np.allclose(a.pose.q, b.pose.q, atol=1e-12) and np.allclose(a.pose.t, b.pose.t, atol=1e-12)
            and abs(a.score - b.score) <= 1e-9 * max(1.0, abs(a.score)))
    bad += not same
    if not same and bad <= 4:
        print("flags", np.array_equal(a.inlier_flags, b.inlier_flags), a.inlier_count, b.inlier_count,
              "score", a.score, b.score, "dq", np.abs(a.pose.q - b.pose.q).max(), "conv", a.converged, b.converged)
  print("mode", md, "mismatching queries", bad, "of", nq, flush=True)
