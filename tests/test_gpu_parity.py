"""GPU parity: the CUDA path (through the C ABI) against golden vectors and the oracle.

Bars (BASELINE.json north_star): identical minimal sets; inlier masks
bit-exact except points within 1e-6 px of the threshold; final pose within
0.01 deg rotation and 1e-4 relative translation.  P3P solutions to 1e-9,
fp32 costs to 1e-5 relative, fp64 MSAC costs to 1e-12 relative.
"""

import math

import numpy as np
import pytest

from oracle import geometry as og
from oracle.posest import Config, errors_sq, msac, ransac
from synth_inputs import batch_a, matches_a

pytestmark = pytest.mark.gpu

INTR_T = (700.0, 700.0, 350.0, 350.0)
TAU = 12.0


@pytest.fixture(scope="module")
def vl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_04185_b200 as vl
    return vl


@pytest.fixture(scope="module")
def intr(vl):
    return vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)


def _near_threshold(q, t, px, X, tol=1e-6):
    """Points whose reprojection error lies within `tol` px of tau under pose (q,t)."""
    e2 = errors_sq(og.q2R(q), t, X, px, INTR_T)
    e = np.sqrt(e2)
    return np.abs(e - TAU) < tol


def _check_mask(flags, ref_flags, q, t, px, X, tol=1e-6):
    diff = flags != ref_flags
    if diff.any():
        amb = _near_threshold(q, t, px, X, tol)
        assert not (diff & ~amb).any(), f"{int((diff & ~amb).sum())} mask differences away from tau"


def _check_pose(q, t, q_ref, t_ref):
    rot = og.rot_err_deg(q, q_ref)
    assert rot < 0.01, rot
    rel = np.linalg.norm(t - t_ref) / max(np.linalg.norm(t_ref), 1e-12)
    assert rel < 1e-4, rel


# ----------------------------------------------------------------------- sampling
def test_sampler_matches_numpy_golden(vl, golden):
    from paper_2601_04185_b200.p3p import sample_minimal_sets
    g = golden("rng")
    for k, (seed, n) in enumerate(zip(g["seeds"], g["n"])):
        s, st = sample_minimal_sets(int(seed), int(n), g["samples"].shape[1])
        assert np.array_equal(s, g["samples"][k]), (seed, n)
        ref = g["states"][k]
        assert st["state"]["state"] == (int(ref[0]) << 64) | int(ref[1])
        assert st["has_uint32"] == int(ref[4]) and st["uinteger"] == int(ref[5])


def test_sampler_chained_batches_match_numpy(vl):
    from paper_2601_04185_b200.p3p import sample_minimal_sets
    for seed, n in [(3, 200_000), (4, 3), (8, 17)]:
        g = np.random.default_rng(seed)
        state = seed
        for _ in range(5):
            ref = np.stack([g.choice(n, 3, replace=False) for _ in range(777)])
            got, state = sample_minimal_sets(state, n, 777)
            assert np.array_equal(got, ref)
        assert state["state"]["state"] == g.bit_generator.state["state"]["state"]


# ----------------------------------------------------------------------- p3p
def test_p3p_matches_reference_golden(vl, golden):
    from paper_2601_04185_b200.p3p import p3p_solve_batch
    g = golden("p3p")
    R, t, idx = p3p_solve_batch(g["bearings"], g["points"])
    assert np.array_equal(idx, g["idx"])
    assert np.abs(R - g["R"]).max() < 1e-9
    assert (np.abs(t - g["t"]).max() / np.abs(g["t"]).max()) < 1e-9


def test_p3p_degenerate_and_scalar(vl):
    from paper_2601_04185_b200.p3p import p3p_solve, p3p_solve_batch
    P = np.array([[0, 0, 2.0], [1, 0, 2.0], [2, 0, 2.0]])
    f = P / np.linalg.norm(P, axis=1, keepdims=True)
    assert p3p_solve(f, P) == []
    R, t, idx = p3p_solve_batch(np.zeros((0, 3, 3)), np.zeros((0, 3, 3)))
    assert R.shape == (0, 3, 3)


# ----------------------------------------------------------------------- msac / refine
def test_msac_matches_reference_golden(vl, intr, golden):
    g = golden("msac")
    for k in range(g["q"].shape[0]):
        pose = vl.Pose(g["q"][k], g["t"][k])
        c, f = vl.msac_score(pose, (g["px"], g["X"], g["w"]), intr, TAU)
        assert math.isclose(c, float(g["costs"][k]), rel_tol=1e-12)
        _check_mask(f, g["flags"][k], g["q"][k], g["t"][k], g["px"], g["X"])


def test_fp32_costs_match_reference_golden(vl, intr, golden):
    """K4 (posest.py:178-220): the estimator's k_score costs of the reference's
    600 golden hypotheses vs the reference's own fp32 costs (score.npz),
    <= 1e-5 relative; every tile shape gives the same bits."""
    from paper_2601_04185_b200.posest import score_hypotheses
    g = golden("score")
    ref = g["costs"]
    got = [score_hypotheses(g["R"], g["t"], g["X"], g["px"], g["w"], intr, float(g["tau"]), shape=s)
           for s in (0, 1, 2)]
    assert np.array_equal(got[0], got[1]) and np.array_equal(got[0], got[2])
    rel = np.abs(got[0] - ref) / np.maximum(np.abs(ref), 1e-30)
    print(f"k_score vs reference fp32 costs: max rel {rel.max():.3e}, median {np.median(rel):.3e}")
    assert rel.max() <= 1e-5, rel.max()
    # ranking: the reference's best hypothesis is the GPU's best too
    assert int(np.argmin(got[0])) == int(np.argmin(ref))


@pytest.mark.parametrize("n,outl", [(10_000, 0.7), (9_999, 0.3), (129, 0.5), (3, 0.0)])
def test_fp32_costs_full_round_vs_oracle(vl, intr, n, outl):
    """One full round's hypotheses (P3P of 1000 samples) over an n_sub-point set
    against the oracle's restatement of _score_hypotheses (pinned to the
    reference by score.npz): <= 1e-5 relative, odd n and single-split sets."""
    from oracle.posest import score_fp32
    from oracle.p3p import p3p_batch
    from oracle.posest import bearings
    from paper_2601_04185_b200.posest import score_hypotheses
    px, X, w, _ = matches_a(n, outl, 1.0, seed=n)
    rng = np.random.default_rng(n)
    smp = np.stack([rng.choice(n, 3, replace=False) for _ in range(300 if n > 3 else 1)])
    f = bearings(px, INTR_T)
    R, t, _ = p3p_batch(f[smp], X[smp])
    if R.shape[0] == 0:
        pytest.skip("degenerate draw")
    ref = score_fp32(R, t, X, px, w, INTR_T, TAU)
    got = score_hypotheses(R, t, X, px, w, intr, TAU)
    assert np.array_equal(got, score_hypotheses(R, t, X, px, w, intr, TAU, shape=2))
    # relative, with a floor of 1e-3 px^2 per unit weight: an exact minimal
    # set (n = 3) has a cost that is pure fp32 rounding noise in both
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3 * w.sum())
    assert rel.max() <= 1e-5, rel.max()


def test_msac_kats(vl, intr):
    pose = vl.Pose.identity()
    xw = np.array([[0.0, 0.0, 2.0], [0.0, 0.0, 3.0]])
    px = np.array([[350.0, 350.0], [360.0, 350.0]])
    c, f = vl.msac_score(pose, (px, xw, np.ones(2)), intr, 5.0)
    assert c == pytest.approx(25.0) and list(f) == [True, False]
    c, f = vl.msac_score(pose, (np.array([[350.0, 350.0]]), np.array([[0, 0, -2.0]]), np.ones(1)),
                         intr, 10.0)
    assert c == pytest.approx(100.0) and not f[0]


def test_refine_matches_reference_golden(vl, intr, golden):
    from paper_2601_04185_b200.refine import CauchyLoss, TruncatedLoss, refine_pose
    g = golden("refine")
    for key in g["cases"]:
        loss = TruncatedLoss(12.0) if str(g[f"{key}_kind"]) == "trunc" else CauchyLoss(12.0)
        r = refine_pose(vl.Pose(g[f"{key}_start_q"], g[f"{key}_start_t"]), g[f"{key}_X"], g[f"{key}_px"],
                        g[f"{key}_w"], loss, intr)
        assert og.rot_err_deg(r.pose.q, g[f"{key}_q"]) < 1e-7
        assert np.linalg.norm(r.pose.t - g[f"{key}_t"]) < 1e-8 * max(1, np.linalg.norm(g[f"{key}_t"]))
        tr = np.array(r.cost_trace)
        ref = g[f"{key}_trace"]
        assert np.all(np.diff(tr) <= 0)
        assert math.isclose(tr[-1], ref[-1], rel_tol=1e-9, abs_tol=1e-9)
        assert r.converged == bool(g[f"{key}_conv"])
        assert abs(r.iterations - int(g[f"{key}_iters"])) <= 1


# ----------------------------------------------------------------------- ransac
def test_ransac_matches_reference_golden(vl, intr, golden):
    g = golden("ransac")
    for k, (n, of, sg, ds, rs, mi, eta) in enumerate(g["cases"]):
        px, X, w, _ = matches_a(int(n), of, sg, seed=int(ds))
        cfg = vl.RansacConfig(seed=int(rs), max_iterations=int(mi), miss_probability=eta)
        e = vl.ransac_pnp((px, X, w), intr, cfg)
        assert e.converged == bool(g[f"r{k}_conv"]), k
        assert e.iterations == int(g[f"r{k}_iters"]), k
        _check_pose(e.pose.q, e.pose.t, g[f"r{k}_q"], g[f"r{k}_t"])
        ref_flags = np.unpackbits(g[f"r{k}_flags"])[: int(n)].astype(bool)
        _check_mask(e.inlier_flags, ref_flags, g[f"r{k}_q"], g[f"r{k}_t"], px, X)
        assert math.isclose(e.score, float(g[f"r{k}_score"]), rel_tol=1e-6, abs_tol=1e-9)


def test_ransac_reference_behaviours(vl, intr):
    """Ports of pkg/tests/test_posest.py:95-175 (same data, same assertions)."""
    q_gt, R_gt, t_gt = og.canon(og.rotvec2q(np.array([0.05, -0.1, 0.2]))), None, np.array([0.1, 0.2, 0.3])
    gt = vl.Pose(q_gt, t_gt)
    px, X, w, _ = matches_a(2000)
    e = vl.ransac_pnp((px, X, w), intr, vl.RansacConfig(seed=5))
    pe = vl.pose_error(e.pose, gt)
    assert e.converged and pe.rotation_error_deg < 1e-6 and pe.translation_error_m < 1e-6
    assert e.iterations == 1000 and e.inlier_count == 2000
    px, X, w, out = matches_a(2000, outlier_frac=0.5, seed=3)
    e = vl.ransac_pnp((px, X, w), intr, vl.RansacConfig(seed=5))
    assert np.array_equal(e.inlier_flags, ~out)
    with pytest.raises(vl.UnderConstrainedError):
        vl.ransac_pnp(matches_a(2)[:3], intr, vl.RansacConfig(seed=0))
    px1 = np.tile(np.array([[350.0, 350.0]]), (5, 1))
    xw1 = np.tile(np.array([[0.0, 0.0, 2.0]]), (5, 1))
    e = vl.ransac_pnp((px1, xw1, np.ones(5)), intr, vl.RansacConfig(seed=0, max_iterations=2000))
    assert not e.converged and e.iterations == 2000
    px, X, w, _ = matches_a(1500, outlier_frac=0.4, sigma=0.5, seed=4)
    a = vl.ransac_pnp((px, X, w), intr, vl.RansacConfig(seed=9))
    b = vl.ransac_pnp((px, X, w), intr, vl.RansacConfig(seed=9))
    assert np.array_equal(a.pose.q, b.pose.q) and np.array_equal(a.pose.t, b.pose.t)
    assert a.score == b.score and np.array_equal(a.inlier_flags, b.inlier_flags)
    matches = [vl.Match2D3D(px[i], X[i], float(w[i]), "e") for i in range(50)]
    assert vl.ransac_pnp(matches, intr, vl.RansacConfig(seed=1)).converged


def test_batch_equals_single_and_oracle(vl, intr):
    pxs, Xs, ws = batch_a(6, 1500, 0.5, 1.0, seed0=40)
    cfg = vl.RansacConfig(seed=0, max_iterations=4000, miss_probability=1e-300)
    seeds = [11 * i + 1 for i in range(6)]
    res = vl.ransac_pnp_batch(list(zip(pxs, Xs, ws)), intr, cfg, seeds=seeds)
    for i in range(6):
        single = vl.ransac_pnp((pxs[i], Xs[i], ws[i]), intr,
                               vl.RansacConfig(seed=seeds[i], max_iterations=4000, miss_probability=1e-300))
        assert np.array_equal(res[i].pose.q, single.pose.q) and np.array_equal(res[i].inlier_flags,
                                                                               single.inlier_flags)
        o = ransac(pxs[i], Xs[i], ws[i], INTR_T, Config(seed=seeds[i], max_iterations=4000,
                                                         miss_probability=1e-300))
        assert res[i].iterations == o.iterations
        _check_pose(res[i].pose.q, res[i].pose.t, o.q, o.t)
        _check_mask(res[i].inlier_flags, o.inlier_flags, o.q, o.t, pxs[i], Xs[i])


def test_host_api_chunked_pipeline_equals_device(vl):
    """ransac_pnp_host (double-buffered H2D/D2H on a copy stream) == one device call."""
    import torch
    from paper_2601_04185_b200.posest import ransac_pnp_device, ransac_pnp_host
    pxs, Xs, ws = batch_a(7, 1200, 0.5, 1.0, seed0=90)
    offsets = np.concatenate([[0], np.cumsum([p.shape[0] for p in pxs])]).astype(np.int64)
    px, X, w = np.concatenate(pxs), np.concatenate(Xs), np.concatenate(ws)
    intr = [vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * 7
    seeds = [3 * i + 2 for i in range(7)]
    cfg = vl.RansacConfig(max_iterations=3000, miss_probability=1e-300)
    ref = ransac_pnp_device(torch.from_numpy(px).cuda(), torch.from_numpy(X).cuda(), torch.from_numpy(w).cuda(),
                            offsets, intr, seeds, cfg)
    ref = {k: v.cpu().numpy() for k, v in ref.items()}
    for chunk in (1, 3, 7, None):  # None: the default staged-admission run
        host, h2d, d2h = ransac_pnp_host(px, X, w, offsets, intr, seeds, cfg, chunk_queries=chunk)
        assert h2d == px.nbytes + X.nbytes + w.nbytes
        for k in ("q", "t", "flags", "count", "score", "iterations", "converged", "stats"):
            assert np.array_equal(host[k], ref[k]), (chunk, k)


@pytest.mark.parametrize("Q,n,batch", [(5000, 24, 1000), (1500, 40, 10_000)])
def test_host_api_above_one_workspace_chunk(vl, Q, n, batch):
    """ransac_pnp_host / ransac_pnp_stream with more queries than one workspace
    chunk (4096 at batch_size 1000, ~646 at 10k) equal ransac_pnp_device
    (which loops over chunks) field by field (vl_capi.cu staged chunks)."""
    import torch
    from paper_2601_04185_b200.posest import ransac_pnp_device, ransac_pnp_host, ransac_pnp_stream
    rng = np.random.default_rng(Q)
    pxs, Xs, ws = [], [], []
    for qi in range(Q):
        px, X, w, _ = matches_a(n, 0.3, 1.0, seed=int(rng.integers(1 << 30)))
        pxs.append(px)
        Xs.append(X)
        ws.append(w)
    offsets = np.arange(Q + 1, dtype=np.int64) * n
    px, X, w = np.concatenate(pxs), np.concatenate(Xs), np.concatenate(ws)
    intr = [vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * Q
    seeds = list(range(Q))
    cfg = vl.RansacConfig(max_iterations=batch, batch_size=batch, miss_probability=1e-300)
    ref = ransac_pnp_device(torch.from_numpy(px).cuda(), torch.from_numpy(X).cuda(), torch.from_numpy(w).cuda(),
                            offsets, intr, seeds, cfg)
    ref = {k: v.cpu().numpy() for k, v in ref.items()}
    host, _, _ = ransac_pnp_host(px, X, w, offsets, intr, seeds, cfg)
    (shost, _, _), = list(ransac_pnp_stream([(torch.from_numpy(px).pin_memory(), torch.from_numpy(X).pin_memory(),
                                              torch.from_numpy(w).pin_memory(), offsets, intr, seeds)], cfg))
    for k in ("q", "t", "flags", "count", "score", "iterations", "converged", "stats"):
        assert np.array_equal(host[k], ref[k]), k
        assert np.array_equal(shost[k], ref[k]), k
    assert ref["converged"].mean() > 0.9


def test_host_stream_equals_device(vl):
    """ransac_pnp_stream (batch k+1's H2D overlapping batch k, first batch staged) == device calls."""
    import torch
    from paper_2601_04185_b200.posest import ransac_pnp_device, ransac_pnp_stream
    cfg = vl.RansacConfig(max_iterations=2000, miss_probability=1e-300)
    batches, refs = [], []
    for b, Q in enumerate((5, 9, 5, 3)):  # sizes change between batches (buffer re-allocation)
        pxs, Xs, ws = batch_a(Q, 900 + 100 * b, 0.5, 1.0, seed0=200 + 10 * b)
        offsets = np.concatenate([[0], np.cumsum([p.shape[0] for p in pxs])]).astype(np.int64)
        px, X, w = np.concatenate(pxs), np.concatenate(Xs), np.concatenate(ws)
        intr = [vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * Q
        seeds = [7 * i + b for i in range(Q)]
        batches.append((torch.from_numpy(px).pin_memory(), torch.from_numpy(X).pin_memory(),
                        torch.from_numpy(w).pin_memory(), offsets, intr, seeds))
        r = ransac_pnp_device(torch.from_numpy(px).cuda(), torch.from_numpy(X).cuda(), torch.from_numpy(w).cuda(),
                              offsets, intr, seeds, cfg)
        refs.append(({k: v.cpu().numpy() for k, v in r.items()}, px.nbytes + X.nbytes + w.nbytes))
    got = list(ransac_pnp_stream(batches, cfg))
    assert len(got) == len(refs)
    for (host, h2d, d2h), (ref, nbytes) in zip(got, refs):
        assert h2d == nbytes and d2h > 0
        for k in ("q", "t", "flags", "count", "score", "iterations", "converged", "stats"):
            assert np.array_equal(host[k], ref[k]), k
    assert list(ransac_pnp_stream([], cfg)) == []
    g = ransac_pnp_stream(batches, cfg)  # a consumer that stops early
    host, _, _ = next(g)
    g.close()
    assert np.array_equal(host["q"], refs[0][0]["q"])


def test_randomized_parity_sweep(vl, intr):
    """40 seeded problems across inlier ratio / noise / size / config regimes:
    GPU ransac_pnp vs the CPU oracle (itself bit-identical to the reference)."""
    rng = np.random.default_rng(2024)
    cases = []
    for k in range(40):
        n = int(rng.choice([50, 300, 1500, 4000, 12000]))
        of = float(rng.choice([0.0, 0.3, 0.5, 0.7, 0.85]))
        sg = float(rng.choice([0.0, 0.5, 1.0, 3.0]))
        mi = int(rng.choice([1000, 3000, 100_000]))
        eta = float(rng.choice([1e-4, 1e-300]))
        cases.append((n, of, sg, 500 + k, 17 * k + 3, mi, eta))
    exact_pose = exact_mask = 0
    for n, of, sg, ds, rs, mi, eta in cases:
        if eta == 1e-300 and mi == 100_000:
            mi = 5000
        px, X, w, _ = matches_a(n, of, sg, seed=ds)
        cfg = vl.RansacConfig(seed=rs, max_iterations=mi, miss_probability=eta)
        e = vl.ransac_pnp((px, X, w), intr, cfg)
        o = ransac(px, X, w, INTR_T, Config(seed=rs, max_iterations=mi, miss_probability=eta))
        assert e.iterations == o.iterations, (n, of, sg, ds, rs)
        assert e.converged == o.converged
        if not o.converged:
            continue
        _check_pose(e.pose.q, e.pose.t, o.q, o.t)
        _check_mask(e.inlier_flags, o.inlier_flags, o.q, o.t, px, X)
        exact_pose += int(og.rot_err_deg(e.pose.q, o.q) < 1e-7)
        exact_mask += int(np.array_equal(e.inlier_flags, o.inlier_flags))
    print(f"sweep: {exact_pose}/40 poses within 1e-7 deg, {exact_mask}/40 masks identical")


def test_hypothesis_split_emulated_ranks_bit_identical(vl, intr):
    """§8e hypothesis-split: G ranks emulated sequentially on one GPU (separate
    contexts; the NCCL SUM all-reduce replaced by a device sum of the ranks'
    partial buffers).  Every rank must end with the single-GPU result, bit-exact."""
    import torch
    from paper_2601_04185_b200 import _lib
    from paper_2601_04185_b200.dist import SplitRun, ransac_pnp_split
    px, X, w, _ = matches_a(6000, 0.6, 1.0, seed=77)
    cfg = vl.RansacConfig(seed=12, max_iterations=4000, miss_probability=1e-300)
    ref = vl.ransac_pnp((px, X, w), intr, cfg)
    assert np.array_equal(ransac_pnp_split((px, X, w), intr, cfg).pose.q, ref.pose.q)  # world = 1
    d = [torch.from_numpy(a).cuda() for a in (px, X, w)]
    for G in (2, 3):
        ctxs = [_lib.Context(0) for _ in range(G)]
        runs = [SplitRun(ctxs[r], d[0], d[1], d[2], [0, px.shape[0]], [intr], [cfg.seed], cfg, r, G)
                for r in range(G)]
        while runs[0].nactive > 0:
            for r in runs:
                r.score()
            total = torch.stack([r.partial for r in runs]).sum(0)
            for r in runs:
                r.partial.copy_(total)
            n = [r.finish() for r in runs]
            assert len(set(n)) == 1
        for r in runs:
            e = r.end()[0]
            assert np.array_equal(e.pose.q, ref.pose.q) and np.array_equal(e.pose.t, ref.pose.t)
            assert np.array_equal(e.inlier_flags, ref.inlier_flags) and e.iterations == ref.iterations


def test_hypothesis_split_argmin_variant(vl, intr):
    """BASELINE's packed (score, index) split: one int64 MIN all-reduce per round
    (emulated ranks on one GPU).  Identical on every rank and for every split
    size; round 1 picks the argmin of the exact fp32 costs; the pose stays close
    to the exact estimator's (it is an approximation of the reference chain)."""
    import torch
    from paper_2601_04185_b200 import _lib
    from paper_2601_04185_b200.dist import SplitRun, ransac_pnp_split
    from paper_2601_04185_b200.geometry import pose_error
    px, X, w, _ = matches_a(6000, 0.6, 1.0, seed=78)
    cfg = vl.RansacConfig(seed=13, max_iterations=4000, miss_probability=1e-300)
    exact = vl.ransac_pnp((px, X, w), intr, cfg)
    one = ransac_pnp_split((px, X, w), intr, cfg, mode="argmin")  # world = 1
    err = pose_error(one.pose, exact.pose)
    assert err.rotation_error_deg < 0.05 and one.converged
    d = [torch.from_numpy(a).cuda() for a in (px, X, w)]
    # round 1: the winning key is the argmin (first minimum) of the full fp32 cost vector
    ref_run = SplitRun(_lib.Context(0), d[0], d[1], d[2], [0, px.shape[0]], [intr], [cfg.seed], cfg, 0, 1)
    ref_run.score()
    ref_run.argmin()
    for G in (2, 3):
        ctxs = [_lib.Context(0) for _ in range(G)]
        runs = [SplitRun(ctxs[r], d[0], d[1], d[2], [0, px.shape[0]], [intr], [cfg.seed], cfg, r, G)
                for r in range(G)]
        first = True
        while runs[0].nactive > 0:
            for r in runs:
                r.score()
                r.argmin()
            keys = torch.stack([r.keys for r in runs]).min(0).values
            if first:
                assert int(keys[0].item()) == int(ref_run.keys[0].item())
                first = False
            for r in runs:
                r.keys.copy_(keys)
            n = [r.finish_argmin() for r in runs]
            assert len(set(n)) == 1
        for r in runs:
            e = r.end()[0]
            assert np.array_equal(e.pose.q, one.pose.q) and np.array_equal(e.pose.t, one.pose.t)
            assert np.array_equal(e.inlier_flags, one.inlier_flags)


@pytest.mark.parametrize("n,kw", [
    (60_000, dict(max_scoring=50_000, max_iterations=2000, miss_probability=1e-300)),  # stride 2, 391 splits
    (3_000, dict(batch_size=1, max_iterations=40, miss_probability=1e-300)),          # one sample per round
    (2_500, dict(batch_size=777, max_iterations=3000, miss_probability=1e-300)),      # odd batch
    (4_000, dict(reproj_threshold=2.5, cauchy_scale=1.0, lm_max_iters=7, max_iterations=2000,
                 miss_probability=1e-300)),
    (3, dict(max_iterations=50, batch_size=50)),                                      # minimal input
    (1_999, dict(max_scoring=997, max_iterations=3000)),                              # odd subset size
])
def test_config_edge_cases_vs_oracle(vl, intr, n, kw):
    """Unusual RansacConfig values and sizes against the CPU oracle."""
    px, X, w, _ = matches_a(n, 0.5 if n > 3 else 0.0, 1.0 if n > 3 else 0.0, seed=n + 5)
    e = vl.ransac_pnp((px, X, w), intr, vl.RansacConfig(seed=4, **kw))
    o = ransac(px, X, w, INTR_T, Config(seed=4, **kw))
    assert e.iterations == o.iterations and e.converged == o.converged
    if o.converged:
        assert og.rot_err_deg(e.pose.q, o.q) < 0.01
        assert np.linalg.norm(e.pose.t - o.t) <= 1e-4 * max(np.linalg.norm(o.t), 1e-9)
        assert (e.inlier_flags != o.inlier_flags).sum() == 0


def test_gpu_concurrent_contexts_from_threads(vl):
    """Two host threads, each with its own library context and stream, estimate
    different query groups at the same time (the serving lanes of
    localize_pipelined): results equal the single-threaded run."""
    import threading

    import torch
    from paper_2601_04185_b200 import _lib
    from paper_2601_04185_b200.posest import ransac_pnp_device
    Q, n = 12, 3000
    qs = [matches_a(n, 0.6, 1.0, seed=900 + i) for i in range(Q)]
    d = [torch.from_numpy(np.concatenate([q[k] for q in qs])).cuda() for k in range(3)]
    offsets = np.arange(Q + 1, dtype=np.int64) * n
    intr = [vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * Q
    seeds = [77 + i for i in range(Q)]
    cfg = vl.RansacConfig(max_iterations=2000)
    ref = {k: v.cpu() for k, v in ransac_pnp_device(d[0], d[1], d[2], offsets, intr, seeds, cfg).items()}
    halves = [(0, Q // 2), (Q // 2, Q)]
    ctxs = [_lib.Context(torch.cuda.current_device()) for _ in halves]
    streams = [torch.cuda.Stream() for _ in halves]
    outs, errs = [None, None], []

    def run(g):
        try:
            a, b = halves[g]
            r0, r1 = int(offsets[a]), int(offsets[b])
            with torch.cuda.stream(streams[g]):
                for _ in range(3):
                    o = ransac_pnp_device(d[0][r0:r1], d[1][r0:r1], d[2][r0:r1], offsets[a:b + 1] - offsets[a],
                                          intr[a:b], seeds[a:b], cfg, ctx=ctxs[g])
                streams[g].synchronize()
                outs[g] = {k: v.cpu() for k, v in o.items()}
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
    th = [threading.Thread(target=run, args=(g,)) for g in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for g, (a, b) in enumerate(halves):
        assert torch.equal(outs[g]["q"], ref["q"][a:b]) and torch.equal(outs[g]["count"], ref["count"][a:b])
        assert torch.equal(outs[g]["flags"], ref["flags"][int(offsets[a]):int(offsets[b])])
