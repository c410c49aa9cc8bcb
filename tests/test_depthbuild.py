"""Dense depth triangulation: oracle pinned to the reference's
goldens; GPU maps / scalar triangulation against the goldens; ports of the
reference's depthbuild unit tests (test_depthbuild.py:36-305).

Parity bar (floating point; arctan2 and summation details differ from numpy
by a few ulp): identical validity masks, z-depth within 1e-6 relative, and
nearly every f32 depth bit-identical to the reference's.
"""

import math
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import depthbuild as od

gpu = pytest.mark.gpu


def _oracle_args(g, p):
    cfg = g[p + "cfg"]
    return (g[p + "targets"], g[p + "conf"], g[p + "scale"], g[p + "R"][0], g[p + "C"][0], g[p + "intr"][0],
            g[p + "R"][1:], g[p + "C"][1:], g[p + "intr"][1:], cfg[0], int(cfg[1]), cfg[2], int(cfg[3]), cfg[4])


def test_oracle_matches_reference_goldens(golden):
    g = golden("depthbuild")
    for i in range(int(g["n"])):
        d, v = od.build_depth_map(*_oracle_args(g, f"c{i}_"))
        np.testing.assert_array_equal(v, g[f"c{i}_valid"])
        np.testing.assert_array_equal(d, g[f"c{i}_depth"])


def _scene_objects(g, p):
    """Entry / covisible namespaces + CorrespondenceFields of a golden case."""
    from paper_2601_04185_b200.geometry import CameraIntrinsics, Pose
    from paper_2601_04185_b200.matchio import CorrespondenceField
    intr = [CameraIntrinsics(r[0], r[1], r[2], r[3], int(r[4]), int(r[5])) for r in g[p + "intr"]]
    poses = [Pose(q, t) for q, t in zip(g[p + "q"], g[p + "t"])]
    for k, ps in enumerate(poses):  # the host pose algebra reproduces the reference's R and centre
        np.testing.assert_array_equal(ps.R, g[p + "R"][k])
        np.testing.assert_array_equal(ps.center(), g[p + "C"][k])
    entry = SimpleNamespace(id="v0", pose=poses[0], intrinsics=intr[0])
    covis = [SimpleNamespace(id=f"v{k}", pose=poses[k], intrinsics=intr[k]) for k in range(1, len(poses))]
    sx, sy = g[p + "scale"]
    fields = [CorrespondenceField("v0", f"v{k + 1}", g[p + "targets"][k], g[p + "conf"][k], sx, sy)
              for k in range(len(covis))]
    return entry, covis, fields


def _cfg(g, p):
    from paper_2601_04185_b200.depthbuild import TriangulationConfig
    c = g[p + "cfg"]
    return TriangulationConfig(angular_threshold_rad=float(c[0]), min_inliers=int(c[1]),
                               confidence_threshold=float(c[2]), max_refine_iters=int(c[3]), refine_tol=float(c[4]))


@gpu
def test_gpu_build_depth_maps_goldens(golden):
    from paper_2601_04185_b200.depthbuild import build_depth_map, build_depth_maps
    g = golden("depthbuild")
    jobs, cfgs = [], []
    same = total = 0
    for i in range(int(g["n"])):
        p = f"c{i}_"
        entry, covis, fields = _scene_objects(g, p)
        dm = build_depth_map(entry, covis, fields, _cfg(g, p))
        ref_d, ref_v = g[p + "depth"], g[p + "valid"]
        np.testing.assert_array_equal(dm.valid, ref_v, err_msg=f"case {i}")
        np.testing.assert_allclose(dm.values[ref_v], ref_d[ref_v], rtol=1e-6, err_msg=f"case {i}")
        assert np.all(dm.values[~ref_v] == 0)
        same += int((dm.values[ref_v].view(np.uint32) == ref_d[ref_v].view(np.uint32)).sum())
        total += int(ref_v.sum())
        jobs.append((entry, covis, fields))
        cfgs.append(_cfg(g, p))
    assert same >= 0.99 * total, f"only {same}/{total} depths bit-identical"
    # batched: jobs sharing a config in one launch give the same maps
    shared = [k for k in range(len(jobs)) if cfgs[k] == cfgs[0]]
    outs = build_depth_maps([jobs[k] for k in shared], cfgs[0])
    for k, dm in zip(shared, outs):
        np.testing.assert_array_equal(dm.valid, g[f"c{k}_valid"])
        single = build_depth_map(*jobs[k], cfgs[0])
        np.testing.assert_array_equal(dm.values, single.values)


@gpu
def test_gpu_triangulate_pixel_goldens(golden):
    """Scalar path (triangulate_pixel / depth_hypothesis) on every cell of the noisy scene."""
    from paper_2601_04185_b200.depthbuild import Observation, depth_hypothesis, triangulate_pixel
    g = golden("depthbuild")
    p = "c2_"
    entry, covis, fields = _scene_objects(g, p)
    cfg = _cfg(g, p)
    grid = fields[0].grid_w
    sx, sy = entry.intrinsics.width / grid, entry.intrinsics.height / grid
    sd, sn, sh = g[p + "scalar_depth"], g[p + "scalar_count"], g[p + "scalar_hyp"]
    k = 0
    for row in range(grid):
        for col in range(grid):
            obs = [Observation(c.pose, c.intrinsics, f.targets[row, col], float(f.confidence[row, col]))
                   for c, f in zip(covis, fields)
                   if f.confidence[row, col] >= cfg.confidence_threshold and f.confidence[row, col] > 0]
            px = np.array([(col + 0.5) * sx, (row + 0.5) * sy])
            kk = np.array([(px[0] - entry.intrinsics.cx) / entry.intrinsics.fx,
                           (px[1] - entry.intrinsics.cy) / entry.intrinsics.fy, 1.0])
            ray = entry.pose.R.T @ (kk / np.linalg.norm(kk))
            r = triangulate_pixel(ray, entry.pose.center(), obs, cfg)
            if sn[k] == 0:
                assert r is None
            else:
                assert r is not None and r[1] == sn[k]
                assert abs(r[0] - sd[k]) <= 1e-7 * sd[k]  # line-search stop is refine_tol = 1e-8 relative
            for j, o in enumerate(obs[:2]):
                h = depth_hypothesis(ray, entry.pose.center(), o)
                if np.isnan(sh[k][j]):
                    assert h is None
                else:
                    assert h == pytest.approx(sh[k][j], rel=1e-9)  # cancellation near parallel rays
            k += 1


@gpu
def test_gpu_random_scenes_vs_oracle():
    """Randomized synthetic rigs (random poses, planar scene, noise + outliers) against the oracle."""
    from paper_2601_04185_b200.depthbuild import TriangulationConfig, build_depth_maps
    from paper_2601_04185_b200.geometry import CameraIntrinsics, Pose, rotvec_to_quat
    from paper_2601_04185_b200.matchio import CorrespondenceField
    rng = np.random.default_rng(7)
    jobs, args = [], []
    cfg = TriangulationConfig()
    for case in range(6):
        V = int(rng.choice([3, 9, 17, 33, 70]))
        gh, gw = int(rng.integers(8, 30)), int(rng.integers(8, 30))
        W = H = 200
        intr = CameraIntrinsics(150.0, 150.0, 100.0, 100.0, W, H)
        ref = Pose(np.array([1.0, 0, 0, 0]), np.zeros(3))
        poses = [Pose(rotvec_to_quat(rng.normal(scale=0.05, size=3)), rng.normal(scale=0.4, size=3))
                 for _ in range(V)]
        # plane z = 4 + 0.1 x seen by the reference; project cell rays into each view
        cols, rows = np.meshgrid(np.arange(gw), np.arange(gh))
        u = (cols + 0.5) * (W / gw)
        v = (rows + 0.5) * (H / gh)
        ray = np.stack([(u - 100) / 150, (v - 100) / 150, np.ones_like(u, dtype=float)], -1)
        z = 4.0 / (1 - 0.1 * ray[..., 0])
        Xw = ray * z[..., None]
        tg, cf = [], []
        for ps in poses:
            xc = Xw @ ps.R.T + ps.t
            t = np.stack([150 * xc[..., 0] / xc[..., 2] + 100, 150 * xc[..., 1] / xc[..., 2] + 100], -1)
            t += rng.normal(scale=0.5, size=t.shape)
            out = rng.random((gh, gw)) < 0.3
            t[out] = rng.uniform(0, 200, size=(out.sum(), 2))
            c = rng.uniform(0.0, 1.0, size=(gh, gw))
            c[rng.random((gh, gw)) < 0.1] = 0.0
            t[c == 0] = np.nan
            tg.append(t)
            cf.append(c)
        entry = SimpleNamespace(id="r", pose=ref, intrinsics=intr)
        covis = [SimpleNamespace(id=f"c{k}", pose=ps, intrinsics=intr) for k, ps in enumerate(poses)]
        fields = [CorrespondenceField("r", f"c{k}", tg[k], cf[k], W / gw, H / gh) for k in range(V)]
        jobs.append((entry, covis, fields))
        irow = [150.0, 150.0, 100.0, 100.0, W, H]
        args.append((np.stack(tg), np.stack(cf), None, ref.R, ref.center(), irow, np.stack([p.R for p in poses]),
                     np.stack([p.center() for p in poses]), [irow] * V))
    outs = build_depth_maps(jobs, cfg)
    for dm, a in zip(outs, args):
        d, v = od.build_depth_map(*a, cfg.angular_threshold_rad, cfg.min_inliers, cfg.confidence_threshold,
                                  cfg.max_refine_iters, cfg.refine_tol)
        np.testing.assert_array_equal(dm.valid, v)
        np.testing.assert_allclose(dm.values[v], d[v], rtol=1e-6)


# ---- ports of the reference's unit tests (test_depthbuild.py:36-305) --------
def _intr(f=100.0, c=50.0, size=100):
    from paper_2601_04185_b200.geometry import CameraIntrinsics
    return CameraIntrinsics(f, f, c, c, size, size)


def _obs_for_point(world_point, center, intr=None, conf=1.0):
    from paper_2601_04185_b200.depthbuild import Observation
    from paper_2601_04185_b200.geometry import Pose
    intr = intr or _intr()
    pose = Pose(np.array([1.0, 0, 0, 0]), -np.asarray(center, dtype=float))
    xc = pose.apply(world_point)
    px = np.array([intr.fx * xc[0] / xc[2] + intr.cx, intr.fy * xc[1] / xc[2] + intr.cy])
    return Observation(pose, intr, px, conf)


def _exact_setup(rng, n_obs, point=None):
    point = np.array([0.3, -0.2, 3.0]) if point is None else point
    obs = []
    for k in range(n_obs):
        ang = 2 * math.pi * k / max(n_obs, 1)
        center = np.array([math.cos(ang), math.sin(ang), 0.0]) * 0.8
        obs.append(_obs_for_point(point, center, conf=float(rng.uniform(0.5, 1.0))))
    return point / np.linalg.norm(point), obs, float(np.linalg.norm(point))


@gpu
def test_gpu_reference_triangulation_ports():
    from paper_2601_04185_b200.depthbuild import (Observation, TriangulationConfig, depth_hypothesis,
                                                  triangulate_pixel)
    from paper_2601_04185_b200.geometry import Pose
    z = np.array([0.0, 0.0, 1.0])
    # test_analytic_two_ray_case (:36-40)
    d = depth_hypothesis(z, np.zeros(3), _obs_for_point(np.array([0.0, 0.0, 2.0]), [1.0, 0.0, 0.0]))
    assert d == pytest.approx(2.0, abs=1e-12)
    # test_parallel_rays_return_none (:42-49)
    obs = Observation(Pose(np.array([1.0, 0, 0, 0]), np.array([0.0, 0.0, 1.0])), _intr(), np.array([50.0, 50.0]),
                      1.0)
    assert depth_hypothesis(z, np.zeros(3), obs) is None
    # test_negative_depth_returns_none (:51-55)
    assert depth_hypothesis(-z, np.zeros(3), _obs_for_point(np.array([0.0, 0.0, 2.0]), [1.0, 0.0, 0.0])) is None
    # test_random_exact_geometry (:57-70)
    rng = np.random.default_rng(0)
    for _ in range(200):
        point = np.array([rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(2, 6)])
        center = rng.normal(size=3) * 0.5
        if abs(center[0]) + abs(center[1]) < 1e-3:
            continue
        d = depth_hypothesis(point / np.linalg.norm(point), np.zeros(3), _obs_for_point(point, center))
        assert d is not None
        np.testing.assert_allclose(d, np.linalg.norm(point), rtol=1e-9)
    cfg = TriangulationConfig()
    # test_five_exact_observations (:82-89)
    ray, obs, gt = _exact_setup(np.random.default_rng(1), 5)
    out = triangulate_pixel(ray, np.zeros(3), obs, cfg)
    assert out is not None and out[1] == 5 and abs(out[0] - gt) / gt < 1e-9
    # test_outliers_rejected_by_voting (:91-102)
    ray, obs, gt = _exact_setup(np.random.default_rng(2), 4)
    for k in range(3):
        pose = Pose(np.array([1.0, 0, 0, 0]), -np.array([0.5 - 0.3 * k, 0.7, 0.0]))
        obs.append(Observation(pose, _intr(), np.array([5.0 + 30 * k, 90.0]), 0.2))
    out = triangulate_pixel(ray, np.zeros(3), obs, cfg)
    assert out is not None and out[1] == 4 and abs(out[0] - gt) / gt < 1e-9
    # test_three_exact_observations_rejected (:104-108)
    ray, obs, _ = _exact_setup(np.random.default_rng(3), 3)
    assert triangulate_pixel(ray, np.zeros(3), obs, cfg) is None
    # test_refinement_reduces_weighted_cost_under_noise (:110-122)
    rng = np.random.default_rng(4)
    ray, obs, gt = _exact_setup(rng, 8)
    noisy = [Observation(o.pose, o.intrinsics, o.target_px + rng.normal(0, 0.5, 2), o.confidence) for o in obs]
    out = triangulate_pixel(ray, np.zeros(3), noisy, cfg)
    assert out is not None and out[1] == 8 and abs(out[0] - gt) / gt < 0.02
    # test_tie_break_keeps_lowest_hypothesis_index (:124-141)
    p_near, p_far = np.array([0.0, 0.0, 2.0]), np.array([0.0, 0.0, 4.0])
    obs = [_obs_for_point(p_near, [1.0, 0.0, 0.0]), _obs_for_point(p_near, [0.0, 1.0, 0.0]),
           _obs_for_point(p_far, [-1.0, 0.0, 0.0]), _obs_for_point(p_far, [0.0, -1.0, 0.0])]
    out = triangulate_pixel(z, np.zeros(3), obs, TriangulationConfig(min_inliers=2))
    assert out is not None and out[1] == 2 and out[0] == pytest.approx(2.0, rel=1e-9)
    assert triangulate_pixel(z, np.zeros(3), [], cfg) is None


def test_config_and_pairing_checks():
    from paper_2601_04185_b200.depthbuild import TriangulationConfig, _check_job
    with pytest.raises(ValueError):
        TriangulationConfig(angular_threshold_rad=0.0)
    with pytest.raises(ValueError):
        TriangulationConfig(min_inliers=0)
    from paper_2601_04185_b200.matchio import CorrespondenceField
    entry = SimpleNamespace(id="a", intrinsics=_intr())
    covis = [SimpleNamespace(id="b"), SimpleNamespace(id="c")]
    f = [CorrespondenceField("a", "b", np.zeros((10, 10, 2)), np.zeros((10, 10)), 10.0, 10.0),
         CorrespondenceField("a", "c", np.zeros((10, 10, 2)), np.zeros((10, 10)), 10.0, 10.0)]
    _check_job(entry, covis, f)
    with pytest.raises(ValueError, match="does not pair"):
        _check_job(entry, covis[::-1], f)
    with pytest.raises(ValueError, match="at least one"):
        _check_job(entry, [], [])
    with pytest.raises(ValueError, match="fields for"):
        _check_job(entry, covis[:1], f)
    bad = [CorrespondenceField("a", "b", np.zeros((10, 10, 2)), np.zeros((10, 10)), 9.0, 10.0)]
    with pytest.raises(ValueError, match="does not span"):
        _check_job(entry, covis[:1], bad)


def test_select_covisible_matches_retrieval_order():
    from paper_2601_04185_b200.depthbuild import select_covisible
    from paper_2601_04185_b200.retrieval import DescriptorIndex
    rng = np.random.default_rng(0)
    vmap = SimpleNamespace(entries=[SimpleNamespace(id=f"e{i}", descriptor=rng.normal(size=8).astype(np.float32))
                                    for i in range(6)])
    assert sorted(e.id for e in select_covisible(vmap.entries[0], SimpleNamespace(entries=vmap.entries[:3]), 50)) \
        == ["e1", "e2"]
    for e in vmap.entries:
        assert e.id not in [c.id for c in select_covisible(e, vmap, 10)]
    got = [e.id for e in select_covisible(vmap.entries[0], vmap, 3)]
    idx = DescriptorIndex.from_entries((e.id, e.descriptor) for e in vmap.entries[1:])
    assert got == [i for i, _ in idx.topk(vmap.entries[0].descriptor.astype(np.float64), 3)]
