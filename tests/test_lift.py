"""Depth lifting / localize parity.

Golden scene (``tests/golden/lift.npz``) = the reference's own synth plane
scene, lift outputs for f64 / f32 fields x GT f32 / dequantised depth, and
reference ``localize`` results.  CPU tests pin the oracle; GPU tests run the
CUDA path (``vl_lift`` + ``vl_ransac_pnp``) against the same fixtures.
"""

import math

import numpy as np
import pytest

from oracle import geometry as og
from oracle import lift as ol
from oracle.posest import errors_sq
from scene_io import unpack_scene

THR = 0.05


def _case(z, k):
    j, i, dk, fdt = (int(v) for v in z[f"L{k}_meta"])
    p = f"s_j{j}_"
    fids = list(z[p + "fids"])
    eid = z["s_entry_ids"][i]
    fk = fids.index(eid)
    fl = {}
    for tag in ("q2db", "db2q"):
        t, c, s = z[f"{p}f{fk}_{tag}_t"], z[f"{p}f{fk}_{tag}_c"], z[f"{p}f{fk}_{tag}_s"]
        if fdt == 1:
            t, c = t.astype(np.float32), c.astype(np.float32)
        fl[tag] = (t, c, float(s[0]), float(s[1]))
    e = f"s_e{i}_"
    intr = z[e + "intr"]
    if dk == 0:
        vals, valid = z[f"gt{i}_values"], z[f"gt{i}_valid"]
    else:
        qp = z[e + "qparams"]
        vals, valid = ol.dequantize(z[e + "codes"], qp[0], qp[1], int(qp[2]))
    return j, i, dk, fdt, fl, intr, vals, valid, z[e + "q"], z[e + "t"]


def test_oracle_lift_matches_reference(golden):
    z = golden("lift")
    for k in range(int(z["nlift"])):
        j, i, dk, fdt, fl, intr, vals, valid, q, t = _case(z, k)
        px, X, w = ol.lift(fl["db2q"], fl["q2db"], vals, valid, intr[:4], intr[4:6], og.q2R(q), t, THR)
        assert np.array_equal(px, z[f"L{k}_px"]) and np.array_equal(w, z[f"L{k}_w"]), k
        assert np.array_equal(X, z[f"L{k}_X"]), k


def test_oracle_dequantize_kats():
    v, ok = ol.dequantize(np.array([[0, 1, 255]], dtype=np.uint8), 0.25, 128.0, 255)
    assert not ok[0, 0] and v[0, 0] == 0.0
    assert v[0, 1] == np.float32(0.25) and v[0, 2] == np.float32(128.0)


def test_oracle_interp_kats():
    # test_localizer.py:34-58 values
    vals = np.array([[1.0, 3.0], [1.0, 3.0]], dtype=np.float32)
    ok = np.ones((2, 2), dtype=bool)
    d, o = ol.interp(vals, ok, np.array([[0.75, 1.0]]))
    assert o[0] and d[0] == pytest.approx(1.5)
    d, o = ol.interp(vals, ok, np.array([[0.4, 1.0]]))
    assert not o[0]


# ----------------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def vl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_04185_b200.localizer as L
    return L


@pytest.mark.gpu
def test_gpu_lift_matches_reference(vl, golden):
    from paper_2601_04185_b200.geometry import CameraIntrinsics, Pose
    z = golden("lift")
    worst = 0.0
    for k in range(int(z["nlift"])):
        j, i, dk, fdt, fl, intr, vals, valid, q, t = _case(z, k)

        class Entry:
            pass

        e = Entry()
        e.id = str(z["s_entry_ids"][i])
        e.pose = Pose(q, t)
        e.intrinsics = CameraIntrinsics(*[float(a) for a in intr[:4]], int(intr[4]), int(intr[5]))
        if dk == 1:
            qp = z[f"s_e{i}_qparams"]
            depth = vl.QuantizedDepthMap(z[f"s_e{i}_codes"], float(qp[0]), float(qp[1]), int(qp[2]), e.intrinsics)
        else:
            depth = vl.DepthMap(vals, valid, e.intrinsics)
        qi = z[f"s_j{j}_intr"]
        job = vl.QueryJob("q", CameraIntrinsics(*[float(a) for a in qi[:4]], int(qi[4]), int(qi[5])),
                          np.zeros(4), {e.id: vl.FieldPair(
                              vl.CorrespondenceField("a", "b", fl["q2db"][0], fl["q2db"][1], *fl["q2db"][2:]),
                              vl.CorrespondenceField("a", "b", fl["db2q"][0], fl["db2q"][1], *fl["db2q"][2:]))})
        px, X, w = (a.cpu().numpy() for a in vl.lift_arrays(job, e, depth, THR))
        assert np.array_equal(px, z[f"L{k}_px"]), k      # pixels and weights are copies: exact
        assert np.array_equal(w, z[f"L{k}_w"]), k
        assert X.shape == z[f"L{k}_X"].shape
        worst = max(worst, float(np.abs(X - z[f"L{k}_X"]).max(initial=0.0)))
    assert worst < 1e-13  # fp64 matmul order only (ulp level)


@pytest.mark.gpu
def test_gpu_lift_object_api(vl, golden):
    from paper_2601_04185_b200.geometry import CameraIntrinsics, Pose
    z = golden("lift")
    vmap, jobs = unpack_scene(z)
    e = vmap.entries[0]
    ms = vl.lift(jobs[0], e, e.qdepth, THR)
    assert len(ms) == int(z["L2_w"].shape[0])  # case 2 = job 0, entry 0, dequantised depth, f64
    assert ms[0].entry_id == e.id and ms[0].weight > 0


@pytest.mark.gpu
def test_gpu_localize_matches_reference(vl, golden):
    from paper_2601_04185_b200.posest import RansacConfig
    z = golden("lift")
    vmap, jobs = unpack_scene(z)
    from parity_util import check_mask
    res = vl.localize_batch(jobs, vmap, RansacConfig(), seeds=[100 + j for j in range(len(jobs))])
    plan = vl.LiftPlan(jobs, vmap)  # the lifted correspondences localize estimated from
    start, end = plan.lift()
    for j, est in enumerate(res):
        assert est.converged == bool(z[f"loc{j}_conv"])
        assert est.iterations == int(z[f"loc{j}_iters"])
        assert og.rot_err_deg(est.pose.q, z[f"loc{j}_q"]) < 0.01
        assert np.linalg.norm(est.pose.t - z[f"loc{j}_t"]) < 1e-4 * max(1e-9, np.linalg.norm(z[f"loc{j}_t"]))
        ref = z[f"loc{j}_flags"]
        assert est.inlier_flags.shape == ref.shape
        px = plan.px[int(start[j]):int(end[j])].cpu().numpy()
        X = plan.X[int(start[j]):int(end[j])].cpu().numpy()
        I = jobs[j].intrinsics
        check_mask(est.inlier_flags, ref, est.pose.q, est.pose.t, px, X, (I.fx, I.fy, I.cx, I.cy), 12.0,
                   q_ref=z[f"loc{j}_q"], t_ref=z[f"loc{j}_t"])
        assert math.isclose(est.score, float(z[f"loc{j}_score"]), rel_tol=1e-6, abs_tol=1e-9)
    single = vl.localize(jobs[1], vmap, RansacConfig(seed=101))
    assert np.array_equal(single.inlier_flags, res[1].inlier_flags)


@pytest.mark.gpu
def test_gpu_gate_interp_decode(vl):
    from paper_2601_04185_b200.geometry import CameraIntrinsics
    rng = np.random.default_rng(0)
    conf = rng.uniform(0, 1, (17, 23)).astype(np.float32)
    conf[conf < 0.2] = 0
    tg = rng.uniform(0, 100, (17, 23, 2)).astype(np.float32)
    f = vl.CorrespondenceField("a", "b", tg, conf, 2.0, 3.0)
    src, tgt, c, idx = vl.filter_matches_arrays(f, 0.3)
    r_src, r_tgt, r_c, r_idx = ol.gate(tg, conf, 2.0, 3.0, 0.3)
    assert np.array_equal(src, r_src) and np.array_equal(tgt, r_tgt) and np.array_equal(c, r_c)
    assert np.array_equal(idx, r_idx)
    intr = CameraIntrinsics(1.0, 1.0, 0.0, 0.0, 23, 17)
    vals = rng.uniform(0.5, 5, (17, 23)).astype(np.float32)
    valid = rng.random((17, 23)) > 0.1
    pts = rng.uniform(-1, 25, (500, 2))
    d, ok = vl.interp_depth_many(vl.DepthMap(np.where(valid, vals, 0), valid, intr), pts)
    rd, rok = ol.interp(np.where(valid, vals, 0), valid, pts)
    assert np.array_equal(ok, rok) and np.array_equal(d, rd)
    assert vl.interp_depth(vl.DepthMap(np.array([[1.0, 3.0], [1.0, 3.0]]), np.ones((2, 2), bool),
                                       CameraIntrinsics(1.0, 1.0, 0.0, 0.0, 2, 2)), (0.75, 1.0)) == pytest.approx(1.5)
    codes = rng.integers(0, 256, (9, 11)).astype(np.uint8)
    dm = vl.dequantize_depth(vl.QuantizedDepthMap(codes, 0.25, 128.0, 255, CameraIntrinsics(1, 1, 0, 0, 11, 9)))
    rv, rvalid = ol.dequantize(codes, 0.25, 128.0, 255)
    assert np.array_equal(dm.values, rv) and np.array_equal(dm.valid, rvalid)
    with pytest.raises(ValueError):
        vl.filter_matches_arrays(f, 1.5)


@pytest.mark.gpu
def test_gpu_filter_matches_cases(vl):
    """The reference's filter_matches cases (test_matchio.py:167-232) through the GPU gate."""
    from paper_2601_04185_b200.matchio import filter_matches
    f = vl.CorrespondenceField("a", "b", np.array([[[np.nan, np.nan], [5.0, 6.0]]]), np.array([[0.0, 0.3]]))
    out = filter_matches(f, 0.0)  # confidence 0 is the no-match sentinel even at threshold 0
    assert len(out) == 1 and np.array_equal(out[0].target_px, [5.0, 6.0])
    f = vl.CorrespondenceField("a", "b", np.zeros((1, 3, 2)), np.array([[0.04, 0.05, 0.9]]))
    assert len(filter_matches(f, 0.05)) == 2  # inclusive threshold
    f = vl.CorrespondenceField("a", "b", np.zeros((2, 2, 2)), np.ones((2, 2)), scale_x=10.0, scale_y=4.0)
    assert [tuple(m.source_px) for m in filter_matches(f, 0.5)] == [(5.0, 2.0), (15.0, 2.0), (5.0, 6.0), (15.0, 6.0)]
    rng = np.random.default_rng(5)
    for _ in range(20):
        conf = rng.random((7, 5))
        conf[rng.random((7, 5)) < 0.3] = 0
        f = vl.CorrespondenceField("a", "b", rng.normal(size=(7, 5, 2)), conf)
        thr = float(rng.random())
        got = filter_matches(f, thr)
        assert len(got) == int(np.sum((conf >= thr) & (conf > 0)))
        _, _, _, cells = vl.filter_matches_arrays(f, thr)
        assert np.all(np.diff(cells) > 0)  # row-major
    with pytest.raises(ValueError):
        filter_matches(f, -0.1)
    with pytest.raises(ValueError):
        filter_matches(f, 1.1)
