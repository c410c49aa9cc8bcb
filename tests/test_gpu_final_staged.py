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


_PLAIN = {}


def _case(vl, n):
    intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
    pxs, Xs, ws = batch_a(160, n, 0.5, 1.0, seed0=n)
    qs = list(zip(pxs, Xs, ws))
    cfg = vl.RansacConfig(max_iterations=2000, miss_probability=1e-300)
    if n not in _PLAIN:
        _PLAIN[n] = _run(vl, "0", qs, cfg, intr)
    return qs, cfg, intr, _PLAIN[n]


# modes (VISLOC_FINAL_STAGED bits): 1 = first pass staged + fused compaction,
# 2 = final pass staged (writes the returned flags / count / score), 3 = both
# (the production default), 7 = both with the debug direct-read path.  n odd
# gives odd per-query offsets (the a0 = even-rounded start); n = 1, 2 mod 512
# leave a 1- or 2-point last chunk.
@pytest.mark.parametrize("mode", ["1", "2", "3", "7"])
@pytest.mark.parametrize("n", [777, 1024, 3001, 513, 1026])
def test_staged_final_equals_plain(vl, n, mode):
    qs, cfg, intr, plain = _case(vl, n)
    staged = _run(vl, mode, qs, cfg, intr)
    for a, b in zip(plain, staged):
        assert a.converged == b.converged
        assert a.inlier_count == b.inlier_count
        assert np.array_equal(a.inlier_flags, b.inlier_flags)
        assert np.allclose(a.pose.q, b.pose.q, rtol=0, atol=1e-12)
        assert np.allclose(a.pose.t, b.pose.t, rtol=0, atol=1e-12)
        assert abs(a.score - b.score) <= 1e-12 * abs(a.score)


@pytest.mark.parametrize("i", [7, 8])
def test_default_final_vs_oracle(vl, i):
    """The production launch (no knob: mode 3 for a > 74-query batch) against the CPU oracle."""
    from parity_util import check_mask, check_pose
    intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
    pxs, Xs, ws = batch_a(160, 777, 0.5, 1.0, seed0=777)
    assert "VISLOC_FINAL_STAGED" not in os.environ
    est = vl.ransac_pnp_batch(list(zip(pxs, Xs, ws)), intr, vl.RansacConfig(max_iterations=2000,
                                                                            miss_probability=1e-300),
                              seeds=list(range(160)))[i]
    ref = ransac(pxs[i], Xs[i], ws[i], (700.0, 700.0, 350.0, 350.0),
                 Config(seed=i, max_iterations=2000, miss_probability=1e-300))
    check_pose(est.pose.q, est.pose.t, ref.q, ref.t)
    check_mask(est.inlier_flags, ref.inlier_flags, est.pose.q, est.pose.t, pxs[i], Xs[i],
               (700.0, 700.0, 350.0, 350.0), 12.0, q_ref=ref.q, t_ref=ref.t)
    assert est.iterations == ref.iterations and est.stats["lo_calls"] == ref.lo_calls
