"""k_final's TMA-streamed full-set pass with the fused inlier compaction.

Batches of more than 74 queries launch k_final with one CTA per query, which
takes the staged path (`msac_full_staged`, vl_ransac.cu); smaller batches use
clusters and plain loads.  The staged path must reproduce the plain one
(posest.py:284-299: full-set MSAC, X[flags_full] in point order, Cauchy LM,
final MSAC): same flags, counts and pose, and scores equal up to fp64
summation order (odd query offsets shift the per-thread point assignment).
One case is also checked against the CPU oracle.
"""

import os

import numpy as np
import pytest

from oracle import geometry as og
from oracle.posest import Config, ransac
from synth_inputs import batch_a

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_04185_b200 as vl
    return vl


def _run(vl, mode, qs, cfg, intr):
    old = os.environ.get("VISLOC_FINAL_STAGED")
    os.environ["VISLOC_FINAL_STAGED"] = mode
    try:
        return vl.ransac_pnp_batch(qs, intr, cfg, seeds=list(range(len(qs))))
    finally:
        if old is None:
            del os.environ["VISLOC_FINAL_STAGED"]
        else:
            os.environ["VISLOC_FINAL_STAGED"] = old


@pytest.mark.parametrize("n", [777, 1024, 3001])
def test_staged_final_equals_plain(vl, n):
    intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
    pxs, Xs, ws = batch_a(160, n, 0.5, 1.0, seed0=n)
    qs = list(zip(pxs, Xs, ws))
    cfg = vl.RansacConfig(max_iterations=2000, miss_probability=1e-300)
    plain = _run(vl, "0", qs, cfg, intr)
    staged = _run(vl, "1", qs, cfg, intr)
    for a, b in zip(plain, staged):
        assert a.converged == b.converged
        assert a.inlier_count == b.inlier_count
        assert np.array_equal(a.inlier_flags, b.inlier_flags)
        assert np.allclose(a.pose.q, b.pose.q, rtol=0, atol=1e-12)
        assert np.allclose(a.pose.t, b.pose.t, rtol=0, atol=1e-12)
        assert abs(a.score - b.score) <= 1e-12 * abs(a.score)
    # default launch (staged) against the CPU oracle on one query
    i = 7
    ref = ransac(pxs[i], Xs[i], ws[i], (700.0, 700.0, 350.0, 350.0),
                 Config(seed=i, max_iterations=2000, miss_probability=1e-300))
    assert og.rot_err_deg(staged[i].pose.q, ref.q) < 0.01
    assert np.linalg.norm(staged[i].pose.t - ref.t) < 1e-4 * np.linalg.norm(ref.t)
