"""Exact scoring pruning (vl_set_scoring_pruning) changes no output bit.

In a round with a best pose the fp32 MSAC sum of every hypothesis is formed
over a prefix of the scoring subset first; a prefix >= the best cost proves
the ordered scan (`costs[h] < best_cost`, posest.py:258) rejects it, so only
the other hypotheses are scored to the end (k_score_tail).  These tests run
the same batches with pruning on and off and require identical poses,
masks, scores and counters, check that pruning actually skipped work, that a
query with a negative weight is never pruned, and compare pruned runs with
the CPU oracle.
"""

import numpy as np
import pytest

from oracle.posest import Config, ransac
from parity_util import check_mask, check_pose
from synth_inputs import matches_a, random_pose

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_04185_b200 as vl
    return vl


def _batch(Q, n, outlier, seed0, neg_weight_q=()):
    qs = []
    for qi in range(Q):
        rng = np.random.default_rng(seed0 + qi)
        _, R, t = random_pose(rng, 0.2, 0.2)
        px, X, w, _ = matches_a(n, outlier, 1.0, seed=seed0 + 7919 * qi + 1, R=R, t=t)
        if qi in neg_weight_q:
            w = w.copy()
            w[18] = -0.25  # (index 18: in the stride-2 scoring subset of n = 20k)
        qs.append((px, X, w))
    return qs


def _run(vl, qs, cfg, seeds, prune):
    import torch
    from paper_2601_04185_b200 import _lib
    from paper_2601_04185_b200.posest import ransac_pnp_device
    ctx = _lib.context()
    ctx.set_pruning(prune)
    ctx.scoring_counters(reset=True)
    try:
        Q = len(qs)
        offsets = np.concatenate([[0], np.cumsum([len(q[0]) for q in qs])]).astype(np.int64)
        d = [torch.from_numpy(np.concatenate([x[k] for x in qs])).cuda() for k in range(3)]
        intr = [vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * Q
        out = {k: v.cpu().numpy() for k, v in ransac_pnp_device(d[0], d[1], d[2], offsets, intr, seeds, cfg).items()}
        return out, ctx.scoring_counters(reset=True)
    finally:
        ctx.set_pruning(True)


def _same(a, b):
    assert set(a) == set(b)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("n,outlier,iters,eta", [
    (50_000, 0.7, 5_000, 1e-300),   # C3 shape (n_sub 10k, 20 split groups), fixed samples
    (9_999, 0.6, 4_000, 1e-300),    # odd n_sub, partial last split
    (9_999, 0.85, 20_000, 1e-4),    # adaptive stop after a few rounds (queries leave at different rounds)
    (30_011, 0.85, 6_000, 1e-300),  # stride 4 subset, low inlier ratio
])
def test_pruning_identical_outputs(vl, n, outlier, iters, eta):
    Q = 40  # coarse scoring items (pruning runs only there)
    qs = _batch(Q, n, outlier, 6100 + n % 97)
    seeds = [77_000 + qi for qi in range(Q)]
    cfg = vl.RansacConfig(max_iterations=iters, miss_probability=eta)
    on, (skipped, tail) = _run(vl, qs, cfg, seeds, True)
    off, (skipped0, tail0) = _run(vl, qs, cfg, seeds, False)
    _same(on, off)
    assert skipped0 == 0 and tail0 == 0
    nominal = int(on["stats"][:, 2].sum())
    assert skipped > 0 and skipped + tail < nominal
    if outlier <= 0.7:
        assert skipped > 0.3 * nominal, (skipped, nominal)


def test_negative_weight_query_not_pruned(vl):
    """A negative weight breaks the monotone prefix: that query is scored in full
    (identical outputs), the others are still pruned."""
    Q, n = 24, 20_000
    qs = _batch(Q, n, 0.7, 8800, neg_weight_q=(3,))
    seeds = [5_000 + qi for qi in range(Q)]
    cfg = vl.RansacConfig(max_iterations=3_000, miss_probability=1e-300)
    on, (skipped, _) = _run(vl, qs, cfg, seeds, True)
    off, _ = _run(vl, qs[:], cfg, seeds, False)
    _same(on, off)
    assert skipped > 0
    # the negative-weight query alone: nothing to skip
    one, (skipped1, tail1) = _run(vl, [qs[3]] * 16, cfg, [seeds[3]] * 16, True)
    assert skipped1 == 0 and tail1 == 0
    # (batches of other sizes run the LO in other cluster shapes: poses agree to ~1e-15)
    assert int(one["iterations"][0]) == int(on["iterations"][3])
    assert np.allclose(one["q"][0], on["q"][3], rtol=0, atol=1e-12)
    assert np.allclose(one["t"][0], on["t"][3], rtol=0, atol=1e-12)
    assert np.array_equal(one["flags"][:n], on["flags"][3 * n:4 * n])


def test_pruned_batch_vs_oracle(vl):
    """Pruned batch (C3 shape, 3 rounds) against the CPU oracle on its first queries."""
    Q, n = 32, 50_000
    qs = _batch(Q, n, 0.7, 9100)
    seeds = [31_000 + qi for qi in range(Q)]
    cfg = vl.RansacConfig(max_iterations=3_000, miss_probability=1e-300)
    on, (skipped, _) = _run(vl, qs, cfg, seeds, True)
    assert skipped > 0
    for qi in range(3):
        px, X, w = qs[qi]
        ref = ransac(px, X, w, (700.0, 700.0, 350.0, 350.0), Config(seed=seeds[qi], max_iterations=3_000,
                                                                     miss_probability=1e-300))
        assert int(on["iterations"][qi]) == ref.iterations
        assert int(on["stats"][qi, 0]) == ref.lo_calls
        check_pose(on["q"][qi], on["t"][qi], ref.q, ref.t)
        check_mask(on["flags"][qi * n:(qi + 1) * n].astype(bool), ref.inlier_flags, on["q"][qi], on["t"][qi],
                   px, X, (700.0, 700.0, 350.0, 350.0), 12.0, q_ref=ref.q, t_ref=ref.t)


def test_pruning_staged_host_api_identical(vl):
    """The staged host pipeline (queries admitted stage by stage, each admission
    followed by a split head / rest round) gives the same results with pruning
    on and off, and the same as the device-resident call."""
    from paper_2601_04185_b200 import _lib
    from paper_2601_04185_b200.posest import ransac_pnp_host
    Q, n = 48, 30_000
    qs = _batch(Q, n, 0.7, 9900)
    seeds = [12_000 + qi for qi in range(Q)]
    cfg = vl.RansacConfig(max_iterations=3_000, miss_probability=1e-4)
    offsets = np.arange(Q + 1, dtype=np.int64) * n
    intr = [vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * Q
    px, X, w = (np.concatenate([x[k] for x in qs]) for k in range(3))
    ctx = _lib.context()
    outs = []
    try:
        for prune in (True, False):
            ctx.set_pruning(prune)
            ctx.scoring_counters(reset=True)
            res, _, _ = ransac_pnp_host(px, X, w, offsets, intr, seeds, cfg, stage_ends=[8, 24, 48])
            outs.append((res, ctx.scoring_counters(reset=True)))
    finally:
        ctx.set_pruning(True)
    (on, (skipped, _)), (off, (skipped0, _)) = outs
    # stages are admitted as their copies land (timing-dependent round
    # compositions, hence LO cluster shapes): decisions exact, poses to ~1e-15
    for k in ("flags", "count", "iterations", "converged", "stats"):
        assert np.array_equal(on[k], off[k]), k
    for k in ("q", "t", "score"):
        assert np.allclose(on[k], off[k], rtol=1e-12, atol=1e-12), k
    assert skipped > 0 and skipped0 == 0
    dev, _ = _run(vl, qs, cfg, seeds, True)
    for k in ("iterations", "converged"):
        assert np.array_equal(on[k], dev[k]), k
    for k in ("q", "t", "score"):  # (other round compositions: LO cluster shapes differ, ~1e-15)
        assert np.allclose(on[k], dev[k], rtol=1e-12, atol=1e-12), k


def test_pruning_mixed_batch_identical(vl):
    """A coarse batch mixing query sizes — single-split subsets (n = 50, nothing to
    prune), a degenerate query whose points are all identical (no P3P solution,
    no hypotheses in any round), odd sizes — gives identical outputs with pruning
    on and off."""
    sizes = [50, 20_000, 77, 9_999, 30_000, 120, 20_000, 15_001] * 5
    qs = []
    for qi, n in enumerate(sizes):
        rng = np.random.default_rng(4400 + qi)
        _, R, t = random_pose(rng, 0.2, 0.2)
        px, X, w, _ = matches_a(n, 0.6, 1.0, seed=4400 + 7919 * qi + 1, R=R, t=t)
        if qi == 9:  # degenerate: every correspondence the same
            px, X = np.repeat(px[:1], n, 0), np.repeat(X[:1], n, 0)
        qs.append((px, X, w))
    seeds = [900 + qi for qi in range(len(qs))]
    cfg = vl.RansacConfig(max_iterations=4_000, miss_probability=1e-300)
    on, (skipped, _) = _run(vl, qs, cfg, seeds, True)
    off, _ = _run(vl, qs, cfg, seeds, False)
    _same(on, off)
    assert skipped > 0
    assert int(on["stats"][9, 1]) == 0 and not on["converged"][9]  # no hypotheses at all
