"""Ports of the reference's own hot-path unit tests, run against the GPU path.

Each test restates an assertion of ``pkg/tests/test_p3p.py``,
``test_refine.py``, ``test_localizer.py`` or ``test_mapstore.py`` (cited per
test) with the same data model and tolerances, calling
``paper_2601_04185_b200`` instead of ``visloc``.
"""

import math

import numpy as np
import pytest

from oracle import geometry as og
from oracle import refine as oref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_04185_b200 as vl
    return vl


def _normalize(v):
    v = np.asarray(v, dtype=np.float64)
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _instance(rng, vl):
    """test_p3p.py:11-19"""
    w = rng.normal(size=3)
    w = w / np.linalg.norm(w) * rng.uniform(0, 0.9 * math.pi)
    gt = vl.Pose(og.rotvec2q(w), rng.normal(size=3))
    xc = np.stack([rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 3), rng.uniform(1.0, 5.0, 3)], axis=-1)
    xw = (xc - gt.t) @ gt.R
    return _normalize(xc), xw, gt


def _contains_gt(vl, R, t, gt):
    for i in range(R.shape[0]):
        pe = vl.pose_error(vl.Pose.from_rt(R[i], t[i]), gt)
        if pe.rotation_error_deg < math.degrees(1e-6) and pe.translation_error_m < 1e-6:
            return True
    return False


# ------------------------------------------------------------------ p3p (test_p3p.py)
def test_p3p_thousand_instances_recover_and_satisfy_contract(vl):
    """test_p3p.py:36-63: all 1000 contain GT; every solution reprojects < 1e-8 rad; <= 4."""
    from paper_2601_04185_b200.p3p import BEARING_TOL, p3p_solve_batch
    rng = np.random.default_rng(1)
    inst = [_instance(rng, vl) for _ in range(1000)]
    f = np.stack([i[0] for i in inst])
    P = np.stack([i[1] for i in inst])
    R, t, s = p3p_solve_batch(f, P)
    misses = 0
    for k in range(1000):
        sel = np.nonzero(s == k)[0]
        assert sel.size <= 4
        if not _contains_gt(vl, R[sel], t[sel], inst[k][2]):
            misses += 1
        for j in sel:
            pred = _normalize(P[k] @ R[j].T + t[j])
            ang = np.arctan2(np.linalg.norm(np.cross(pred, f[k]), axis=-1), np.sum(pred * f[k], axis=-1))
            assert ang.max() < BEARING_TOL
    assert misses == 0


def test_p3p_degenerate_inputs_give_empty(vl):
    """test_p3p.py:66-77"""
    from paper_2601_04185_b200.p3p import p3p_solve
    pts = np.array([[0.0, 0.0, 2.0], [0.0, 0.0, 3.0], [0.0, 0.0, 4.0]])
    assert p3p_solve(_normalize(pts), pts) == []
    pts = np.array([[0.1, 0.2, 2.0], [0.2, 0.4, 4.0], [0.3, 0.6, 6.0]])
    assert p3p_solve(_normalize(pts), pts) == []
    pts = np.array([[0.5, 0.1, 2.0], [0.5, 0.1, 2.0], [0.0, -0.4, 3.0]])
    b = _normalize(np.array([[0.1, 0.0, 1.0], [0.3, 0.2, 1.0], [0.0, -0.1, 1.0]]))
    assert p3p_solve(b, pts) == []


def test_p3p_batch_matches_scalar(vl):
    """test_p3p.py:80-95 (atol 1e-12)"""
    from paper_2601_04185_b200.p3p import p3p_solve, p3p_solve_batch
    rng = np.random.default_rng(4)
    inst = [_instance(rng, vl) for _ in range(50)]
    R, t, s = p3p_solve_batch(np.stack([i[0] for i in inst]), np.stack([i[1] for i in inst]))
    for k in range(50):
        scalar = p3p_solve(inst[k][0], inst[k][1])
        idx = np.nonzero(s == k)[0]
        assert len(scalar) == len(idx)
        for sol, bi in zip(scalar, idx):
            np.testing.assert_allclose(sol.R, R[bi], atol=1e-12)
            np.testing.assert_allclose(sol.t, t[bi], atol=1e-12)


# ------------------------------------------------------------------ refine (test_refine.py)
INTR_R = (500.0, 470.0, 320.0, 240.0)


def _problem(rng, vl, n=80, pix_noise=0.0):
    """test_refine.py:22-33"""
    pose = vl.Pose(og.rotvec2q(rng.normal(size=3) * 0.4), rng.normal(size=3) * 0.3)
    xc = np.stack([rng.uniform(-1.2, 1.2, n), rng.uniform(-1.0, 1.0, n), rng.uniform(2.0, 6.0, n)], axis=-1)
    xw = (xc - pose.t) @ pose.R
    px = np.stack([INTR_R[0] * xc[:, 0] / xc[:, 2] + INTR_R[2], INTR_R[1] * xc[:, 1] / xc[:, 2] + INTR_R[3]], -1)
    if pix_noise:
        px = px + rng.normal(0, pix_noise, px.shape)
    return pose, xw, px


@pytest.fixture(scope="module")
def intr_r(vl):
    return vl.CameraIntrinsics(500.0, 470.0, 320.0, 240.0, 640, 480)


def test_jacobian_matches_central_differences(vl, intr_r):
    """test_refine.py:37-52: analytic Jacobian vs central differences, rel err < 1e-4."""
    from paper_2601_04185_b200.refine import apply_delta, pose_jacobian, pose_residuals
    rng = np.random.default_rng(0)
    worst = 0.0
    for _ in range(20):
        pose, xw, px = _problem(rng, vl, n=20, pix_noise=2.0)
        J = pose_jacobian(pose, xw, intr_r)
        h = 1e-6
        Jfd = np.zeros_like(J)
        for k in range(6):
            d = np.zeros(6)
            d[k] = h
            rp, _ = pose_residuals(apply_delta(pose, d), xw, px, intr_r)
            rm, _ = pose_residuals(apply_delta(pose, -d), xw, px, intr_r)
            Jfd[:, :, k] = (rp - rm) / (2 * h)
        worst = max(worst, float(np.abs(J - Jfd).max() / np.abs(Jfd).max()))
    assert worst < 1e-4


def test_jacobian_behind_rows_zeroed_and_robust_cost(vl, intr_r):
    """test_refine.py:54-59, :146-161"""
    from paper_2601_04185_b200.refine import CauchyLoss, TruncatedLoss, pose_jacobian, robust_cost
    J = pose_jacobian(vl.Pose.identity(), np.array([[0.0, 0.0, 2.0], [0.0, 0.0, -2.0]]), intr_r)
    assert np.abs(J[0]).max() > 0 and np.abs(J[1]).max() == 0
    xw = np.array([[0.0, 0.0, -1.0]])
    c = robust_cost(vl.Pose.identity(), xw, np.array([[320.0, 240.0]]), np.array([2.0]), TruncatedLoss(3.0), intr_r)
    assert c == pytest.approx(18.0)
    c = robust_cost(vl.Pose.identity(), xw, np.array([[320.0, 240.0]]), np.array([1.0]), CauchyLoss(3.0), intr_r)
    assert math.isinf(c)


def test_refine_stationary_recovers_monotone(vl, intr_r):
    """test_refine.py:84-128"""
    from paper_2601_04185_b200.refine import CauchyLoss, TruncatedLoss, apply_delta, refine_pose
    rng = np.random.default_rng(1)
    pose, xw, px = _problem(rng, vl)
    r = refine_pose(pose, xw, px, np.ones(len(xw)), CauchyLoss(12.0), intr_r)
    pe = vl.pose_error(r.pose, pose)
    assert r.converged and pe.rotation_error_deg < 1e-10 and pe.translation_error_m < 1e-12
    rng = np.random.default_rng(2)
    pose, xw, px = _problem(rng, vl, n=200)
    start = apply_delta(pose, np.array([0.006, -0.005, 0.007, 0.03, -0.02, 0.04]))
    assert vl.pose_error(start, pose).rotation_error_deg > 0.3
    r = refine_pose(start, xw, px, np.ones(200), CauchyLoss(12.0), intr_r)
    pe = vl.pose_error(r.pose, pose)
    assert pe.rotation_error_deg < math.degrees(1e-8) and pe.translation_error_m < 1e-8
    rng = np.random.default_rng(3)
    pose, xw, px = _problem(rng, vl, n=200)
    start = apply_delta(pose, np.array([0.004, 0.003, -0.002, -0.02, 0.01, 0.02]))
    r = refine_pose(start, xw, px, np.ones(200), TruncatedLoss(12.0), intr_r)
    assert vl.pose_error(r.pose, pose).translation_error_m < 1e-8
    rng = np.random.default_rng(4)
    pose, xw, px = _problem(rng, vl, n=300, pix_noise=1.5)
    start = apply_delta(pose, np.array([0.01, -0.01, 0.005, 0.05, 0.02, -0.04]))
    r = refine_pose(start, xw, px, rng.uniform(0.3, 1.0, 300), CauchyLoss(6.0), intr_r)
    assert all(b <= a for a, b in zip(r.cost_trace, r.cost_trace[1:]))


def test_refine_weight_scale_and_outliers(vl, intr_r):
    """test_refine.py:120-144"""
    from paper_2601_04185_b200.refine import CauchyLoss, apply_delta, refine_pose
    rng = np.random.default_rng(5)
    pose, xw, px = _problem(rng, vl, n=150, pix_noise=1.0)
    start = apply_delta(pose, np.array([0.004, 0.002, -0.006, 0.02, -0.03, 0.01]))
    w = rng.uniform(0.2, 1.0, 150)
    a = refine_pose(start, xw, px, w, CauchyLoss(8.0), intr_r)
    b = refine_pose(start, xw, px, 7.3 * w, CauchyLoss(8.0), intr_r)
    assert np.abs(a.pose.q - b.pose.q).max() < 1e-9 and np.abs(a.pose.t - b.pose.t).max() < 1e-9
    rng = np.random.default_rng(6)
    pose, xw, px = _problem(rng, vl, n=400)
    out = rng.random(400) < 0.25
    px = px.copy()
    px[out] = rng.uniform(0, 640, (int(out.sum()), 2))
    start = apply_delta(pose, np.array([0.003, -0.002, 0.004, 0.02, 0.01, -0.02]))
    r = refine_pose(start, xw, px, np.ones(400), CauchyLoss(6.0), intr_r)
    pe = vl.pose_error(r.pose, pose)
    assert pe.rotation_error_deg < 0.05 and pe.translation_error_m < 0.01
    with pytest.raises(ValueError):
        refine_pose(vl.Pose.identity(), np.zeros((2, 3)), np.zeros((2, 2)), np.ones(2), CauchyLoss(1.0), intr_r)


def test_refine_trace_matches_oracle(vl, intr_r):
    """LM trajectory parity: GPU cost trace vs the oracle's, step by step."""
    from paper_2601_04185_b200.refine import CauchyLoss, apply_delta, refine_pose
    rng = np.random.default_rng(11)
    pose, xw, px = _problem(rng, vl, n=500, pix_noise=1.0)
    start = apply_delta(pose, np.array([0.01, -0.008, 0.006, 0.04, -0.03, 0.02]))
    w = rng.uniform(0.3, 1.0, 500)
    r = refine_pose(start, xw, px, w, CauchyLoss(6.0), intr_r)
    o_pose, o_conv, o_it, o_trace = oref.refine((start.q, start.t), xw, px, w, oref.CAUCHY, 6.0, INTR_R)
    assert r.iterations == o_it and r.converged == o_conv
    np.testing.assert_allclose(r.cost_trace, o_trace, rtol=1e-10)
    assert og.rot_err_deg(r.pose.q, o_pose[0]) < 1e-8


# ------------------------------------------------------------------ lift helpers (test_localizer / test_mapstore)
def test_interp_depth_kats(vl):
    """test_localizer.py:34-58"""
    from paper_2601_04185_b200.localizer import DepthMap, interp_depth
    I2 = vl.CameraIntrinsics(1.0, 1.0, 0.0, 0.0, 2, 2)
    dm = DepthMap(np.array([[2.0, 2.0], [3.0, 3.0]]), np.ones((2, 2), bool), I2)
    assert interp_depth(dm, (1.0, 1.0)) == pytest.approx(2.5)
    bad = np.ones((2, 2), bool)
    bad[1, 1] = False
    assert interp_depth(DepthMap(np.array([[2.0, 2.0], [3.0, 3.0]]) * bad, bad, I2), (1.0, 1.0)) is None
    dm = DepthMap(np.array([[1.0, 4.0], [1.0, 4.0]]), np.ones((2, 2), bool), I2)
    assert interp_depth(dm, (0.5, 0.5)) == pytest.approx(1.0)
    assert interp_depth(dm, (1.5, 1.5)) == pytest.approx(4.0)
    assert interp_depth(dm, (0.4, 1.0)) is None and interp_depth(dm, (1.6, 1.0)) is None
    dm = DepthMap(np.array([[1.0, 3.0], [1.0, 3.0]]), np.ones((2, 2), bool), I2)
    assert interp_depth(dm, (0.75, 1.0)) == pytest.approx(1.5)


def test_dequantize_kats(vl):
    """test_mapstore.py:46-72: codes 1 -> d_min, 255 -> d_max, 0 invalid, round trip."""
    from paper_2601_04185_b200.localizer import QuantizedDepthMap, dequantize_depth
    I = vl.CameraIntrinsics(1.0, 1.0, 0.0, 0.0, 4, 1)
    dm = dequantize_depth(QuantizedDepthMap(np.array([[0, 1, 128, 255]], np.uint8), 0.25, 128.0, 255, I))
    assert not dm.valid[0, 0] and dm.values[0, 0] == 0.0
    assert dm.values[0, 1] == pytest.approx(0.25) and dm.values[0, 3] == pytest.approx(128.0, rel=1e-6)
    assert dm.values[0, 2] == pytest.approx(0.25 * math.sqrt(512.0), rel=1e-6)
    codes = np.arange(1, 256, dtype=np.uint8)[None]
    dm = dequantize_depth(QuantizedDepthMap(codes, 0.25, 128.0, 255, vl.CameraIntrinsics(1.0, 1.0, 0.0, 0.0, 255, 1)))
    span = math.log(128.0) - math.log(0.25)
    back = 1 + np.floor((np.log(dm.values.astype(np.float64)) - math.log(0.25)) / span * 254 + 0.5)
    assert np.array_equal(back.astype(np.uint8), codes)


def test_lift_span_check_and_threshold_errors(vl, golden):
    """test_localizer.py:114-129 span check -> ValueError; threshold outside [0,1]."""
    from scene_io import unpack_scene
    from paper_2601_04185_b200.localizer import CorrespondenceField, FieldPair, QueryJob, lift
    z = golden("lift")
    vmap, jobs = unpack_scene(z)
    e = vmap.entries[0]
    job = jobs[0]
    fp = job.fields[e.id]
    bad = CorrespondenceField("a", "b", fp.db_to_query.targets, fp.db_to_query.confidence,
                              fp.db_to_query.scale_x * 2, fp.db_to_query.scale_y)
    job2 = QueryJob(job.query_id, job.intrinsics, job.descriptor, {e.id: FieldPair(fp.query_to_db, bad)})
    with pytest.raises(ValueError):
        lift(job2, e, e.qdepth)
    with pytest.raises(ValueError):
        lift(job, e, e.qdepth, threshold=1.5)


def test_localize_retrieval_and_seed_invariance(vl, golden):
    """test_localizer.py:166-186: retrieval order does not matter; seeds move the pose < 1e-9 on exact data."""
    from scene_io import unpack_scene
    from paper_2601_04185_b200.localizer import localize
    z = golden("lift")
    vmap, jobs = unpack_scene(z)
    cfg = vl.RansacConfig(seed=4)
    a = localize(jobs[0], vmap, cfg)

    class Rev:
        def __init__(self, entries):
            self.entries = list(reversed(entries))
    b = localize(jobs[0], Rev(vmap.entries), cfg)
    assert np.array_equal(a.pose.q, b.pose.q) and np.array_equal(a.inlier_flags, b.inlier_flags)
