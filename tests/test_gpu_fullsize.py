"""Parity at BASELINE's full problem sizes.

The CPU oracle needs seconds per full-size query, so exact comparisons use a
few queries and the rest of the batch is checked through size-independent
properties: every query of a full C3-shaped batch (50k correspondences,
n_sub = 10k, fixed 10k minimal samples) matches its own single-query run
(batch independence: same decisions and masks, poses to ~1e-15 — the LO
reductions associate by cluster size), recovers its ground-truth pose to the noise level,
finds the true inliers, and the work counters add up; C2-scale (200k
correspondences, stride-20 scoring subset) and C4-scale (ε = 5 %, 100k
minimal samples) single queries match the oracle / the ground truth.
"""

import numpy as np
import pytest

from oracle import geometry as og
from oracle.posest import Config, ransac
from synth_inputs import matches_a, random_pose

pytestmark = pytest.mark.gpu

INTR_T = (700.0, 700.0, 350.0, 350.0)


@pytest.fixture(scope="module")
def vl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_04185_b200 as vl
    return vl


def _query(qi, n, outlier, sigma, seed0):
    rng = np.random.default_rng(seed0 + qi)
    q, R, t = random_pose(rng, 0.2, 0.2)
    px, X, w, out = matches_a(n, outlier, sigma, seed=seed0 + 7919 * qi + 1, R=R, t=t)
    return px, X, w, out, q, t


def test_c3_shaped_batch_full_size(vl):
    """48 queries x 50k correspondences, 30 % inliers, sigma 1 px, 10k minimal samples each."""
    import torch
    from paper_2601_04185_b200.posest import ransac_pnp_device
    Q, n = 48, 50_000
    qs = [_query(qi, n, 0.7, 1.0, 4000) for qi in range(Q)]
    intr = [vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * Q
    seeds = [1_000_003 * 4000 + qi for qi in range(Q)]
    cfg = vl.RansacConfig(max_iterations=10_000, miss_probability=1e-300)
    offsets = np.arange(Q + 1, dtype=np.int64) * n
    d = [torch.from_numpy(np.concatenate([x[k] for x in qs])).cuda() for k in range(3)]
    out = {k: v.cpu().numpy() for k, v in ransac_pnp_device(d[0], d[1], d[2], offsets, intr, seeds, cfg).items()}
    assert np.all(out["iterations"] == 10_000) and np.all(out["converged"] == 1)
    stats = out["stats"]  # lo_calls, hypotheses, evaluations, rounds
    assert np.all(stats[:, 3] == 10) and np.all(stats[:, 0] >= 1)
    assert np.array_equal(stats[:, 2], stats[:, 1] * 10_000)  # n_sub = 10k: evals = hypotheses x n_sub
    for qi, (px, X, w, outl, gq, gt) in enumerate(qs):
        rot = og.rot_err_deg(out["q"][qi], gq)
        assert rot < 0.05, (qi, rot)
        assert np.linalg.norm(out["t"][qi] - gt) < 5e-3 * max(1.0, np.linalg.norm(gt))
        flags = out["flags"][offsets[qi]:offsets[qi + 1]].astype(bool)
        # true inliers (sigma 1 px, tau 12 px) are all found; few outliers land within tau by chance
        assert flags[~outl].mean() > 0.999
        assert flags[outl].mean() < 0.01
        assert out["count"][qi] == flags.sum()
    # batch independence: two queries re-run alone.  The single query runs its
    # LO / final passes as an 8-CTA cluster (a 48-query batch uses 4), so the
    # fp64 reductions associate differently: same samples, hypotheses, LO
    # decisions and masks; poses equal to ~1e-15
    for qi in (0, Q - 1):
        px, X, w = qs[qi][:3]
        e = vl.ransac_pnp((px, X, w), intr[qi], vl.RansacConfig(seed=seeds[qi], max_iterations=10_000,
                                                                miss_probability=1e-300))
        assert og.rot_err_deg(e.pose.q, out["q"][qi]) < 1e-9
        assert np.allclose(e.pose.t, out["t"][qi], rtol=1e-12, atol=1e-14)
        assert np.array_equal(e.inlier_flags, out["flags"][offsets[qi]:offsets[qi + 1]].astype(bool))
        assert e.stats["lo_calls"] == stats[qi, 0] and e.stats["hypotheses"] == stats[qi, 1]


def test_c3_query_full_size_vs_oracle(vl):
    """One full-size C3 query against the CPU oracle (itself bit-identical to the reference)."""
    px, X, w, _, _, _ = _query(5, 50_000, 0.7, 1.0, 4100)
    cfg = vl.RansacConfig(seed=77, max_iterations=10_000, miss_probability=1e-300)
    e = vl.ransac_pnp((px, X, w), vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700), cfg)
    o = ransac(px, X, w, INTR_T, Config(seed=77, max_iterations=10_000, miss_probability=1e-300))
    assert e.iterations == o.iterations == 10_000
    assert og.rot_err_deg(e.pose.q, o.q) < 0.01
    assert np.linalg.norm(e.pose.t - o.t) <= 1e-4 * np.linalg.norm(o.t)
    assert (e.inlier_flags != o.inlier_flags).sum() == 0


def test_c2_scale_single_query_vs_oracle(vl):
    """200k correspondences (scoring subset = every 20th), 10k minimal samples."""
    px, X, w, _, _, _ = _query(1, 200_000, 0.66, 1.0, 4200)
    cfg = vl.RansacConfig(seed=5, max_iterations=10_000, miss_probability=1e-300)
    e = vl.ransac_pnp((px, X, w), vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700), cfg)
    o = ransac(px, X, w, INTR_T, Config(seed=5, max_iterations=10_000, miss_probability=1e-300))
    assert e.iterations == o.iterations
    assert og.rot_err_deg(e.pose.q, o.q) < 0.01
    assert np.linalg.norm(e.pose.t - o.t) <= 1e-4 * np.linalg.norm(o.t)
    assert (e.inlier_flags != o.inlier_flags).sum() == 0


def test_c4_scale_low_inlier_lo_heavy(vl):
    """10k correspondences, 5 % inliers, 100k minimal samples (fixed): converges to the
    ground truth, runs many LO calls, and the adaptive default stops at the
    reference's required_iterations (73,679 samples at eps = 0.05 ... clamped by
    what the subset shows)."""
    px, X, w, outl, gq, gt = _query(2, 10_000, 0.95, 1.0, 4300)
    intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
    e = vl.ransac_pnp((px, X, w), intr, vl.RansacConfig(seed=9, max_iterations=100_000, miss_probability=1e-300))
    assert e.converged and e.iterations == 100_000
    assert e.stats["lo_calls"] >= 3
    assert og.rot_err_deg(e.pose.q, gq) < 0.1
    assert e.inlier_flags[~outl].mean() > 0.99
    a = vl.ransac_pnp((px, X, w), intr, vl.RansacConfig(seed=9))  # adaptive default (eta = 1e-4)
    eps = a.inlier_count / px.shape[0]
    need = vl.required_iterations(eps, 1e-4)
    assert a.converged and a.iterations <= 100_000
    assert og.rot_err_deg(a.pose.q, gq) < 0.1
    assert need > 10_000  # the low-inlier regime the config is about


def test_million_point_query_vs_oracle(vl):
    """One query with 1M correspondences (subset stride 100, final refinement
    over ~300k inliers, one CTA streaming the full set) against the oracle."""
    from parity_util import check_mask, check_pose
    px, X, w, _ = matches_a(1_000_000, 0.7, 1.0, seed=1234)
    intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
    est = vl.ransac_pnp((px, X, w), intr, vl.RansacConfig(seed=5, max_iterations=2000, miss_probability=1e-300))
    ref = ransac(px, X, w, INTR_T, Config(seed=5, max_iterations=2000, miss_probability=1e-300))
    assert est.converged and est.iterations == ref.iterations == 2000
    assert est.stats["lo_calls"] == ref.lo_calls
    check_pose(est.pose.q, est.pose.t, ref.q, ref.t)
    check_mask(est.inlier_flags, ref.inlier_flags, est.pose.q, est.pose.t, px, X, INTR_T, 12.0, q_ref=ref.q,
               t_ref=ref.t)


def test_mixed_batch_edge_queries_vs_oracle(vl):
    """One batch mixing minimal (n = 3, 4), all-outlier, small and large
    queries: every query behaves as it does alone in the oracle (including the
    in-band failures: converged False, identity pose, inf score)."""
    import math
    from parity_util import check_mask, check_pose
    rng = np.random.default_rng(77)
    qs = []
    for n, outl in ((3, 0.0), (4, 0.0), (500, 1.0), (2000, 0.5), (30_000, 0.7), (7, 0.0), (1200, 0.95)):
        px, X, w, _ = matches_a(n, outl, 0.5, seed=int(rng.integers(1 << 30)))
        qs.append((px, X, w))
    intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
    cfg = vl.RansacConfig(max_iterations=3000, miss_probability=1e-300)
    seeds = list(range(11, 11 + len(qs)))
    ests = vl.ransac_pnp_batch(qs, intr, cfg, seeds=seeds)
    for (px, X, w), est, sd in zip(qs, ests, seeds):
        ref = ransac(px, X, w, INTR_T, Config(seed=sd, max_iterations=3000, miss_probability=1e-300))
        assert est.converged == ref.converged and est.iterations == ref.iterations
        assert est.inlier_count == ref.inlier_count
        if math.isinf(ref.score):
            assert math.isinf(est.score) and np.array_equal(est.pose.q, [1.0, 0.0, 0.0, 0.0])
            continue
        check_pose(est.pose.q, est.pose.t, ref.q, ref.t)
        check_mask(est.inlier_flags, ref.inlier_flags, est.pose.q, est.pose.t, px, X, INTR_T, 12.0, q_ref=ref.q,
                   t_ref=ref.t)
