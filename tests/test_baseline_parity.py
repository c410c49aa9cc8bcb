"""Parity at the BASELINE.json configs, against the REAL reference.

``tests/golden/baseline.npz`` and ``lift_full.npz`` were produced by
``tests/golden/make_golden.py baseline lift_full``, which runs the reference
``ransac_pnp`` / ``lift`` / ``localize`` (``posest.py:223-299``,
``localizer.py:134-238``) on inputs this file regenerates from seeds:

* C1  — generator A, n = 2k, eps = 0.3, 10k fixed minimal samples;
* C4  — generator A, n = 10k, eps = 0.05, 100k fixed samples (LO-heavy) and
        the adaptive default (eta = 1e-4, needed ~ 73.7k);
* C5  — generator B, K = 10 x 117^2 f32 fields, 8-bit log-quantised depth,
        and the fp16-depth variant (reference oracle: DepthMap(values=
        fp16.astype(f32))), default adaptive config;
* C2  — generator B, K = 20 x 83^2 fields, f32 depth, 10k fixed samples.

Bars: iteration counts and the reference's LO-call counts equal; pose within
0.01 deg / 1e-4 relative translation; masks bit-exact except points within
1e-6 px of tau (parity_util.check_mask); lifted matches: count and order
exact, pixels and weights bit-exact (sha256 of the bytes), world points
within 1e-12 m.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from oracle import geometry as og
from parity_util import check_mask, check_pose
from synth_inputs import INTR_A, matches_a

INTR_T = (700.0, 700.0, 350.0, 350.0)
TAU = 12.0
THR = 0.05


def _cases(z):
    names = [str(s) for s in z["names"]]
    return {nm: tuple(z["cases"][i]) for i, nm in enumerate(names)}


def _inputs_a(case):
    n, of, sg, ds, rs, mi, eta = case
    px, X, w, _ = matches_a(int(n), of, sg, seed=int(ds))
    return px, X, w, int(rs), int(mi), float(eta)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _lift_case(z, name):
    from synth_inputs import lifted_scene
    K, g, seed0, mi = (int(v) for v in z[name + "_meta"])
    eta = float(z[name + "_eta"])
    qs = [int(q) for q in z[name + "_queries"]]
    depth = {"c5u8": "u8", "c5f16": "f16", "c2": "f32"}[name]
    vmap, jobs, dc = lifted_scene(K, 0, g, seed=seed0, depth_kind=depth, fields="f32", only=qs)
    return vmap, jobs, dc, qs, seed0, mi, eta


# ----------------------------------------------------------------------------- CPU: the oracle
def test_oracle_c1_matches_reference(golden):
    from oracle.posest import Config, ransac
    z = golden("baseline")
    px, X, w, rs, mi, eta = _inputs_a(_cases(z)["c1"])
    r = ransac(px, X, w, INTR_T, Config(seed=rs, max_iterations=mi, miss_probability=eta))
    assert r.iterations == int(z["c1_iters"]) and r.lo_calls == int(z["c1_lo_calls"])
    assert np.array_equal(r.q, z["c1_q"]) and np.array_equal(r.t, z["c1_t"])
    assert np.array_equal(np.packbits(r.inlier_flags), z["c1_flags"]) and r.score == float(z["c1_score"])


@pytest.mark.parametrize("name", ["c5u8", "c5f16", "c2"])
def test_oracle_lift_full_shapes_match_reference(golden, name):
    """The oracle lift at full C5 / C2 shape reproduces the reference bit for bit (first query)."""
    from oracle import lift as ol
    z = golden("lift_full")
    vmap, jobs, dc, qs, *_ = _lift_case(z, name)
    qi, job = qs[0], jobs[0]
    p = f"{name}_q{qi}_"
    xs = []
    for k, e in enumerate(sorted(vmap.entries, key=lambda e: e.id)):
        fp = job.fields[e.id]
        if dc is not None:
            vals, valid = np.asarray(dc[e.id].values).astype(np.float32), dc[e.id].valid
        else:
            q = e.qdepth
            vals, valid = ol.dequantize(q.codes, q.d_min, q.d_max, q.levels)
        f1 = (fp.db_to_query.targets, fp.db_to_query.confidence, fp.db_to_query.scale_x, fp.db_to_query.scale_y)
        f2 = (fp.query_to_db.targets, fp.query_to_db.confidence, fp.query_to_db.scale_x, fp.query_to_db.scale_y)
        I = e.intrinsics
        px, X, w = ol.lift(f1, f2, vals, valid, (I.fx, I.fy, I.cx, I.cy), (I.width, I.height),
                           og.q2R(e.pose.q), e.pose.t, THR)
        assert px.shape[0] == int(z[p + "count"][k])
        assert _sha(px) == str(z[p + "hpx"][k]) and _sha(w) == str(z[p + "hw"][k])
        xs.append(X[::61])
    assert np.array_equal(np.concatenate(xs), z[p + "Xs"])


# ----------------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def vl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_04185_b200 as vl
    return vl


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c4", "c4a"])
def test_gpu_baseline_config_matches_reference(vl, golden, name):
    """C1 / C4 through the drop-in ransac_pnp vs the reference's own run."""
    from oracle.posest import msac
    z = golden("baseline")
    px, X, w, rs, mi, eta = _inputs_a(_cases(z)[name])
    intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
    est = vl.ransac_pnp((px, X, w), intr, vl.RansacConfig(seed=rs, max_iterations=mi, miss_probability=eta))
    p = name + "_"
    ref_flags = np.unpackbits(z[p + "flags"])[: int(z[p + "n"])].astype(bool)
    print(f"{name}: iterations {est.iterations} (ref {int(z[p + 'iters'])}), LO calls "
          f"{est.stats['lo_calls']} (ref {int(z[p + 'lo_calls'])}), inliers {est.inlier_count} "
          f"(ref {int(z[p + 'count'])})")
    assert est.converged == bool(z[p + "conv"])
    assert est.iterations == int(z[p + "iters"])
    assert est.stats["lo_calls"] == int(z[p + "lo_calls"])
    check_pose(est.pose.q, est.pose.t, z[p + "q"], z[p + "t"])
    check_mask(est.inlier_flags, ref_flags, est.pose.q, est.pose.t, px, X, INTR_T, TAU,
               q_ref=z[p + "q"], t_ref=z[p + "t"])
    # both ways: the reference MSAC (oracle, pinned bit-exact) of the GPU pose
    _, own = msac((est.pose.q, est.pose.t), px, X, w, INTR_T, TAU)
    check_mask(est.inlier_flags, own, est.pose.q, est.pose.t, px, X, INTR_T, TAU)
    assert math.isclose(est.score, float(z[p + "score"]), rel_tol=1e-6)


def _gpu_lift_query(vl, vmap, job, dc):
    """Every entry's lift for one query in localize order (ascending id)."""
    from paper_2601_04185_b200.localizer import lift_arrays
    out = []
    for e in sorted(vmap.entries, key=lambda e: e.id):
        depth = dc[e.id] if dc is not None else e.qdepth
        out.append(tuple(a.cpu().numpy() for a in lift_arrays(job, e, depth, THR)))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c5u8", "c5f16", "c2"])
def test_gpu_lift_full_shapes_match_reference(vl, golden, name):
    """vl_lift at full C5 (u8 codes, fp16 depth) and C2 (f32) shape vs the reference lift."""
    z = golden("lift_full")
    vmap, jobs, dc, qs, *_ = _lift_case(z, name)
    worst = 0.0
    for qi, job in zip(qs, jobs):
        p = f"{name}_q{qi}_"
        lifts = _gpu_lift_query(vl, vmap, job, dc)
        assert [a[0].shape[0] for a in lifts] == [int(c) for c in z[p + "count"]]
        for k, (px, X, w) in enumerate(lifts):
            assert _sha(px) == str(z[p + "hpx"][k]), (qi, k)  # pixels / weights: bit-exact copies
            assert _sha(w) == str(z[p + "hw"][k]), (qi, k)
            assert np.allclose(X.sum(axis=0), z[p + "Xsum"][k], rtol=1e-12, atol=1e-9)
        Xs = np.concatenate([X[::61] for _, X, _ in lifts])
        worst = max(worst, float(np.abs(Xs - z[p + "Xs"]).max()))
    print(f"{name}: max |X - X_ref| = {worst:.2e} m")
    assert worst < 1e-12  # fp64 matmul association only


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c5u8", "c5f16", "c2"])
def test_gpu_localize_full_shapes_match_reference(vl, golden, name):
    """localize_batch (one lift launch sequence + batched estimator) and the
    IMLC serving loop (localize_pipelined over pinned FieldArena payloads)
    vs the reference localize at C5 / C2 shape."""
    from paper_2601_04185_b200.localizer import FieldPair, QueryJob, localize_batch, localize_pipelined
    from paper_2601_04185_b200.matchio import FieldArena, field_bytes
    z = golden("lift_full")
    vmap, jobs, dc, qs, seed0, mi, eta = _lift_case(z, name)
    cfg = vl.RansacConfig(max_iterations=mi, miss_probability=eta)
    seeds = [1_000_003 * seed0 + qi for qi in qs]
    res = localize_batch(jobs, vmap, cfg, seeds=seeds, depth_cache=dc)
    for qi, job, est in zip(qs, jobs, res):
        p = f"{name}_q{qi}_loc_"
        lifts = _gpu_lift_query(vl, vmap, job, dc)
        px = np.concatenate([a[0] for a in lifts])
        X = np.concatenate([a[1] for a in lifts])
        ref_flags = np.unpackbits(z[p + "flags"])[: int(z[p + "n"])].astype(bool)
        print(f"{name} q{qi}: n {px.shape[0]}, iterations {est.iterations} (ref {int(z[p + 'iters'])}), "
              f"LO calls {est.stats['lo_calls']} (ref {int(z[p + 'lo_calls'])}), inliers {est.inlier_count} "
              f"(ref {int(z[p + 'count'])})")
        assert est.converged == bool(z[p + "conv"])
        assert est.iterations == int(z[p + "iters"])
        assert est.stats["lo_calls"] == int(z[p + "lo_calls"])
        check_pose(est.pose.q, est.pose.t, z[p + "q"], z[p + "t"])
        I = job.intrinsics
        check_mask(est.inlier_flags, ref_flags, est.pose.q, est.pose.t, px, X, (I.fx, I.fy, I.cx, I.cy), TAU,
                   q_ref=z[p + "q"], t_ref=z[p + "t"])
        assert math.isclose(est.score, float(z[p + "score"]), rel_tol=1e-6)
    # the same queries with their fields as IMLC payloads in one pinned arena
    order = [(k, eid) for k in range(len(jobs)) for eid in sorted(jobs[k].fields)]
    blobs = []
    for k, eid in order:
        fp = jobs[k].fields[eid]
        blobs += [field_bytes(fp.query_to_db), field_bytes(fp.db_to_query)]
    arena = FieldArena(blobs)
    fields = [{} for _ in jobs]
    for i, (k, eid) in enumerate(order):
        fields[k][eid] = FieldPair(arena[2 * i], arena[2 * i + 1])
    ajobs = [QueryJob(j.query_id, j.intrinsics, j.descriptor, fields[k], j.k_loc) for k, j in enumerate(jobs)]
    pres = localize_pipelined([(ajobs, arena)], vmap, cfg, seeds=seeds, depth_cache=dc)
    for a, b in zip(res, pres):
        assert a.iterations == b.iterations and a.stats == b.stats
        assert np.array_equal(a.pose.q, b.pose.q) and np.array_equal(a.pose.t, b.pose.t)
        assert np.array_equal(a.inlier_flags, b.inlier_flags) and a.score == b.score
