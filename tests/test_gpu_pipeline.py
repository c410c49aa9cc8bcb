"""The pipelined round loop (small batches: round r+1's sampling + P3P on a
side stream while round r is scored and scanned) gives exactly the results
of the plain round loop.

Each configuration runs in two fresh processes, VISLOC_PIPE=1 and
VISLOC_PIPE=0 (the switch is read once per process), and every output
field is compared bit for bit; queries stop at different rounds (adaptive
stop), so the speculative batch of a finished query must never count.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys, json, numpy as np, torch
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/tests"]
import paper_2601_04185_b200 as vl
from paper_2601_04185_b200.posest import ransac_pnp_device
from synth_inputs import matches_a, random_pose
spec = json.loads(sys.argv[2])
qs = []
for qi, (n, outl) in enumerate(spec["queries"]):
    rng = np.random.default_rng(500 + qi)
    _, R, t = random_pose(rng, 0.2, 0.2)
    px, X, w, _ = matches_a(n, outl, 1.0, seed=500 + 7919 * qi + 1, R=R, t=t)
    qs.append((px, X, w))
offsets = np.concatenate([[0], np.cumsum([len(q[0]) for q in qs])]).astype(np.int64)
d = [torch.from_numpy(np.concatenate([x[k] for x in qs])).cuda() for k in range(3)]
intr = [vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * len(qs)
cfg = vl.RansacConfig(max_iterations=spec["iters"], miss_probability=spec["eta"], batch_size=spec["batch"])
out = ransac_pnp_device(d[0], d[1], d[2], offsets, intr, [77 + qi for qi in range(len(qs))], cfg)
np.savez(sys.argv[3], **{k: v.cpu().numpy() for k, v in out.items()})
"""


def _run(spec, pipe, tmp_path):
    f = tmp_path / f"out_{pipe}.npz"
    env = dict(os.environ, VISLOC_PIPE=str(pipe))
    subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), json.dumps(spec), str(f)], env=env, check=True,
                   timeout=600)
    return dict(np.load(f))


@pytest.mark.parametrize("spec", [
    dict(queries=[[2000, 0.7]], iters=10_000, eta=1e-300, batch=1000),            # C1
    dict(queries=[[10_000, 0.95]], iters=20_000, eta=1e-300, batch=1000),         # C4-like
    dict(queries=[[3000, 0.5], [800, 0.8], [20_000, 0.6], [500, 0.9], [5000, 0.3]],
         iters=30_000, eta=1e-4, batch=1000),                                    # adaptive, ragged stops
    dict(queries=[[1500, 0.7], [1501, 0.85]], iters=2_500, eta=1e-300, batch=999),  # partial last batch
    dict(queries=[[3, 0.0], [4, 0.0], [7, 0.3]], iters=1_000, eta=1e-4, batch=250),     # minimal sets
    dict(queries=[[60_000, 0.8], [2_000, 0.5]], iters=7_777, eta=1e-2, batch=250),     # stride-6 subset, many rounds
])
def test_pipelined_loop_identical(spec, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a, b = _run(spec, 1, tmp_path), _run(spec, 0, tmp_path)
    assert set(a) == set(b)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert np.all(a["iterations"] <= spec["iters"])
