"""Generate golden vectors by running the REAL reference (``/root/reference``).

Run in the build container only (the reference does not exist on the GPU
box):  ``python tests/golden/make_golden.py``.  Writes small ``.npz``
fixtures next to this script; they pin the oracle (``tests/test_oracle_golden.py``)
and the GPU path (``tests/test_gpu_*.py``).  numpy version is recorded
because the minimal-sample sets come from numpy's PCG64 stream.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from visloc.geometry import CameraIntrinsics, Pose, rotvec_to_quat  # noqa: E402
from visloc.p3p import p3p_solve_batch  # noqa: E402
from visloc.posest import (RansacConfig, _bearings, _score_hypotheses, msac_score,  # noqa: E402
                           ransac_pnp)
from visloc.refine import CauchyLoss, TruncatedLoss, refine_pose  # noqa: E402

sys.path.insert(0, str(OUT.parent))
sys.path.append(str(OUT.parent.parent))  # repo root (oracle / package types for the synthetic scenes)
from synth_inputs import INTR_A, GT_A, matches_a, refine_problem  # noqa: E402


def rng_vectors():
    cases = [(0, 2000), (5, 3), (5, 4), (7, 50), (11, 23_000), (12345, 200_000), (2**40 + 3, 50_000),
             (99, 2**31 - 1)]
    seeds, ns, samples, states = [], [], [], []
    for seed, n in cases:
        g = np.random.default_rng(seed)
        s = np.stack([g.choice(n, size=3, replace=False) for _ in range(2000)])
        st = g.bit_generator.state
        seeds.append(seed)
        ns.append(n)
        samples.append(s)
        states.append([st["state"]["state"] >> 64, st["state"]["state"] & (2**64 - 1),
                       st["state"]["inc"] >> 64, st["state"]["inc"] & (2**64 - 1),
                       st["has_uint32"], st["uinteger"]])
    np.savez_compressed(OUT / "rng.npz", seeds=np.array(seeds, dtype=np.uint64), n=np.array(ns),
                        samples=np.stack(samples), states=np.array(states, dtype=np.uint64),
                        numpy_version=np.array(np.__version__))


def p3p_vectors():
    px, X, w, _ = matches_a(4000, 0.5, 1.0, seed=21)
    b = _bearings(px, INTR_A)
    rng = np.random.default_rng(3)
    smp = np.stack([rng.choice(4000, 3, replace=False) for _ in range(3000)])
    R, t, idx = p3p_solve_batch(b[smp], X[smp])
    np.savez_compressed(OUT / "p3p.npz", bearings=b[smp], points=X[smp], R=R, t=t, idx=idx)
    return R, t, px, X, w


def score_vectors(R, t, px, X, w):
    sub = slice(0, 4000, 2)
    costs = _score_hypotheses(R[:600], t[:600], X[sub], px[sub], w[sub], INTR_A, 12.0)
    np.savez_compressed(OUT / "score.npz", R=R[:600], t=t[:600], px=px[sub], X=X[sub], w=w[sub],
                        costs=costs, tau=12.0)


def msac_vectors():
    px, X, w, _ = matches_a(3000, 0.4, 2.0, seed=8)
    out = {"px": px, "X": X, "w": w}
    rng = np.random.default_rng(1)
    qs, ts, costs, flags = [], [], [], []
    for k in range(6):
        dq = rotvec_to_quat(rng.normal(size=3) * 0.01 * k)
        pose = Pose(dq, np.zeros(3)).compose(GT_A) if k else GT_A
        pose = Pose(pose.q, pose.t + rng.normal(size=3) * 0.01 * k)
        c, f = msac_score(pose, (px, X, w), INTR_A, 12.0)
        qs.append(pose.q)
        ts.append(pose.t)
        costs.append(c)
        flags.append(f)
    out.update(q=np.array(qs), t=np.array(ts), costs=np.array(costs), flags=np.array(flags))
    np.savez_compressed(OUT / "msac.npz", **out)


def refine_vectors():
    recs = {}
    for k, (kind, n, noise, outl) in enumerate([("trunc", 300, 1.0, 0.3), ("trunc", 2000, 0.5, 0.5),
                                               ("cauchy", 500, 1.0, 0.25), ("cauchy", 3000, 0.3, 0.0)]):
        start, X, px, w = refine_problem(np.random.default_rng(100 + k), n, noise, outl)
        loss = TruncatedLoss(12.0) if kind == "trunc" else CauchyLoss(12.0)
        r = refine_pose(start, X, px, w, loss, INTR_A, max_iters=100)
        recs[f"c{k}"] = dict(kind=kind, start_q=start.q, start_t=start.t, X=X, px=px, w=w, q=r.pose.q,
                             t=r.pose.t, iters=r.iterations, conv=r.converged, trace=np.array(r.cost_trace))
    flat = {}
    for key, d in recs.items():
        for k2, v in d.items():
            flat[f"{key}_{k2}"] = np.asarray(v)
    flat["cases"] = np.array(list(recs))
    np.savez_compressed(OUT / "refine.npz", **flat)


def ransac_vectors():
    cases = [
        # (n, outlier_frac, sigma, data seed, ransac seed, max_iterations, eta)
        (2000, 0.0, 0.0, 0, 5, 100_000, 1e-4),
        (2000, 0.5, 0.0, 3, 5, 100_000, 1e-4),
        (1500, 0.4, 0.5, 4, 9, 100_000, 1e-4),
        (3000, 0.3, 1.0, 9, 3, 100_000, 1e-4),
        (800, 0.3, 0.0, 6, 1, 100_000, 1e-4),
        (2000, 0.7, 1.0, 12, 7, 3000, 1e-300),
        (23_000, 0.2, 0.0, 7, 2, 100_000, 1e-4),
        (12_000, 0.6, 1.0, 13, 17, 2000, 1e-300),
    ]
    flat = {"cases": np.array(cases, dtype=np.float64)}
    for k, (n, of, sg, ds, rs, mi, eta) in enumerate(cases):
        px, X, w, _ = matches_a(int(n), of, sg, seed=int(ds))
        cfg = RansacConfig(seed=int(rs), max_iterations=int(mi), miss_probability=eta)
        e = ransac_pnp((px, X, w), INTR_A, cfg)
        flat[f"r{k}_q"] = e.pose.q
        flat[f"r{k}_t"] = e.pose.t
        flat[f"r{k}_flags"] = np.packbits(e.inlier_flags)
        flat[f"r{k}_score"] = np.array(e.score)
        flat[f"r{k}_iters"] = np.array(e.iterations)
        flat[f"r{k}_conv"] = np.array(e.converged)
        flat[f"r{k}_count"] = np.array(e.inlier_count)
    np.savez_compressed(OUT / "ransac.npz", **flat)


def lift_vectors():
    """Reference lift + localize on a small synthetic plane scene (test_localizer._bench style)."""
    from visloc.depthbuild import DepthMap
    from visloc.localizer import lift, localize
    from visloc.mapbuild import synthetic_posed_entries, synthetic_query_jobs
    from visloc.mapstore import dequantize_depth, quantize_depth
    from visloc.matchio import CorrespondenceField
    from visloc.localizer import FieldPair
    from visloc.synth import NoiseSpec, SceneSpec, make_queries, make_scene
    from scene_io import pack_scene

    f = 70.0
    intr = CameraIntrinsics(f, f, 70.0, 70.0, 140, 140)
    spec = SceneSpec(num_cameras=6, width=140, height=140, camera_spread=0.3, camera_backoff=0.25,
                     rotation_jitter_deg=3.0, seed=21, intrinsics=intr)
    scene = make_scene(spec)
    grid = 32
    entries = synthetic_posed_entries(scene)
    gt = {}
    for i, e in enumerate(entries):
        d, v = scene.gt_depth_grid(i, grid, grid)
        gt[e.id] = DepthMap(d.astype(np.float32), v, intr)
        e.qdepth = quantize_depth(gt[e.id])
    queries = make_queries(scene, 4, 22)
    pairs = synthetic_query_jobs(scene, queries, grid, k_loc=4,
                                 noise=NoiseSpec(sigma_px=1.0, outlier_fraction=0.3), noise_seed=23)
    jobs = [p[0] for p in pairs]

    class _Map:
        pass

    vmap = _Map()
    vmap.entries = entries
    out = pack_scene(entries, jobs)
    for i, e in enumerate(entries):
        out[f"gt{i}_values"], out[f"gt{i}_valid"] = gt[e.id].values, gt[e.id].valid
    # lift per (job, entry): f64 fields x {gt f32 depth, dequantized codes}; f32 fields x gt depth
    k = 0
    for j, job in enumerate(jobs[:1]):
        for i, e in enumerate(entries[:3]):
            for depth_kind in ("gt", "deq"):
                depth = gt[e.id] if depth_kind == "gt" else dequantize_depth(e.qdepth)
                for fdt in ("f64", "f32"):
                    jb = job
                    if fdt == "f32":
                        fp = job.fields[e.id]

                        def c32(fl):
                            return CorrespondenceField(fl.source_id, fl.target_id, fl.targets.astype(np.float32),
                                                       fl.confidence.astype(np.float32), fl.scale_x, fl.scale_y)
                        import copy
                        jb = copy.copy(job)
                        jb.fields = dict(job.fields)
                        jb.fields[e.id] = FieldPair(c32(fp.query_to_db), c32(fp.db_to_query))
                    ms = lift(jb, e, depth, 0.05)
                    out[f"L{k}_meta"] = np.array([j, i, 0 if depth_kind == "gt" else 1, 0 if fdt == "f64" else 1])
                    out[f"L{k}_px"] = np.array([m.query_px for m in ms]).reshape(-1, 2)
                    out[f"L{k}_X"] = np.array([m.world_point for m in ms]).reshape(-1, 3)
                    out[f"L{k}_w"] = np.array([m.weight for m in ms])
                    k += 1
    out["nlift"] = np.array(k)
    for j, job in enumerate(jobs):
        est = localize(job, vmap, RansacConfig(seed=100 + j), depth_cache={})
        out[f"loc{j}_q"], out[f"loc{j}_t"] = est.pose.q, est.pose.t
        out[f"loc{j}_flags"] = est.inlier_flags
        out[f"loc{j}_iters"] = np.array(est.iterations)
        out[f"loc{j}_conv"] = np.array(est.converged)
        out[f"loc{j}_score"] = np.array(est.score)
    np.savez_compressed(OUT / "lift.npz", **out)


def imlc_vectors():
    """Reference read_field on valid and damaged IMLC blobs (matchio.py:158-200)."""
    import json
    import struct
    import tempfile
    from visloc.matchio import CorrespondenceField, FieldFormatError, read_field, write_field

    rng = np.random.default_rng(5)
    h, w = 7, 9
    tg = rng.uniform(0, 140, (h, w, 2)).astype(np.float32)
    cf = rng.uniform(0, 1, (h, w)).astype(np.float32)
    cf[cf < 0.3] = 0.0
    tg[cf == 0.0] = np.nan  # allowed: unmatched cells may carry NaN targets
    good = CorrespondenceField("query_0007", "db_\u00e9ntry_12", tg, cf, 2.5, 3.25)
    tmp = Path(tempfile.mkdtemp())
    write_field(good, tmp / "good.imlc")
    base = (tmp / "good.imlc").read_bytes()
    rec0 = len(base) - 12 * h * w
    cases = {"good": base}
    for cut in (0, 2, 4, 6, 8, 10, 12, 15, 12 + 10 + 2, 12 + 10 + 4 + 3, rec0 - 20, rec0 - 1, rec0, rec0 + 5,
                len(base) - 1):
        cases[f"cut{cut}"] = base[:cut]
    cases["magic"] = b"IMLD" + base[4:]
    cases["version"] = base[:4] + struct.pack("<I", 2) + base[8:]
    cases["trailing"] = base + b"\x00\x01\x02"
    gw_off = rec0 - 24
    cases["zero_grid"] = base[:gw_off] + struct.pack("<II", 0, 3) + base[gw_off + 8:rec0]
    cases["huge_grid"] = base[:gw_off] + struct.pack("<II", 0xFFFFFFFF, 0xFFFFFFFF) + base[gw_off + 8:]

    def with_rec(i, j, k, v):
        b = bytearray(base)
        struct.pack_into("<f", b, rec0 + 12 * (i * w + j) + 4 * k, v)
        return bytes(b)
    cases["conf_gt1"] = with_rec(2, 3, 2, 1.5)
    cases["conf_neg"] = with_rec(0, 0, 2, -0.25)
    cases["conf_nan"] = with_rec(6, 8, 2, float("nan"))
    j0 = int(np.argmax(cf.reshape(-1) > 0))
    cases["target_nan"] = with_rec(j0 // w, j0 % w, 0, float("nan"))
    cases["target_inf"] = with_rec(j0 // w, j0 % w, 1, float("inf"))
    out, names = {}, []
    for i, (name, blob) in enumerate(cases.items()):
        p_ = tmp / f"{i}.imlc"
        p_.write_bytes(blob)
        try:
            fld = read_field(p_)
            exp = {"name": name, "ok": True, "source_id": fld.source_id, "target_id": fld.target_id,
                   "grid_w": fld.grid_w, "grid_h": fld.grid_h, "scale_x": fld.scale_x, "scale_y": fld.scale_y}
            out[f"targets{i}"], out[f"conf{i}"] = fld.targets, fld.confidence
        except FieldFormatError as exc:
            exp = {"name": name, "ok": False, "cls": type(exc).__name__, "msg": str(exc), "offset": exc.offset}
        out[f"blob{i}"] = np.frombuffer(blob, dtype=np.uint8)
        out[f"expect{i}"] = np.array(json.dumps(exp))
        names.append(name)
    out["n"] = np.array(len(names))
    np.savez_compressed(OUT / "imlc.npz", **out)


def retrieval_vectors():
    """Reference DescriptorIndex.topk (retrieval.py:66-82) incl. exact ties and k > size."""
    from visloc.retrieval import DescriptorIndex
    rng = np.random.default_rng(11)
    out = {}
    for tag, E, D in (("a", 300, 16), ("b", 120, 256)):
        vecs = rng.normal(size=(E, D)).astype(np.float32)
        vecs[7] = vecs[3] * 2.0        # identical direction: exact tie, broken by id
        vecs[50] = vecs[3]
        ids = [f"e{(i * 7919) % 1000:04d}" for i in range(E)]  # ids not in insertion order
        idx = DescriptorIndex(D)
        for i in range(E):
            idx.add(ids[i], vecs[i])
        Q = 20
        qs = rng.normal(size=(Q, D))
        qs[0] = vecs[3].astype(np.float64) * 3.0  # ties at the top
        res_ids, res_sims = [], []
        for q in qs:
            r = idx.topk(q, 12)
            res_ids.append([ids.index(e) for e, _ in r])
            res_sims.append([s_ for _, s_ in r])
        out[f"{tag}_vecs"], out[f"{tag}_qs"] = vecs, qs
        out[f"{tag}_ids"] = np.array([int(i[1:]) for i in ids])
        out[f"{tag}_top"], out[f"{tag}_sims"] = np.array(res_ids), np.array(res_sims)
        small = DescriptorIndex(D)
        for i in range(5):
            small.add(ids[i], vecs[i])
        out[f"{tag}_small_top"] = np.array([ids.index(e) for e, _ in small.topk(qs[1], 12)])
    np.savez_compressed(OUT / "retrieval.npz", **out)


def mapstore_vectors():
    """Reference depth codecs (mapstore.py:96-134, :390-425): quantize incl. clip bounds,
    exact-threshold neighbours and invalid pixels; nearest-valid block reduction; requantization."""
    from visloc.depthbuild import DepthMap
    from visloc.mapstore import (QuantizedDepthMap, _downsample_codes_nearest_valid, _requantize_codes,
                                 dequantize_depth, quantize_depth)
    rng = np.random.default_rng(2024)
    intr = CameraIntrinsics(100.0, 100.0, 50.0, 40.0, 100, 80)
    out = {}
    qcases = [(0.25, 128.0, 255), (0.25, 128.0, 65535), (0.5, 40.0, 1000), (0.25, 128.0, 2), (1.0, 2.0, 1),
              (0.1, 300.0, 511), (0.25, 128.0, 31)]
    for i, (dmin, dmax, L) in enumerate(qcases):
        h, w = 37, 53
        vals = np.exp(rng.uniform(np.log(dmin * 0.5), np.log(dmax * 2.0), size=(h, w))).astype(np.float32)
        flat = vals.reshape(-1)
        # exact decode points and their f32 neighbours (quantize(dequantize(c)) == c is the reference claim)
        c = rng.integers(1, L + 1, size=200)
        d = (dmin * np.exp((c - 1.0) / max(L - 1, 1) * math.log(dmax / dmin))).astype(np.float32)
        flat[:200] = d
        flat[200:400] = np.nextafter(d, np.float32(np.inf))
        flat[400:600] = np.nextafter(d, np.float32(0))
        # midpoints between adjacent levels (rounding boundaries) and their neighbours
        cm = rng.integers(1, max(L, 2), size=200)
        dm = (dmin * np.exp((cm - 0.5) / max(L - 1, 1) * math.log(dmax / dmin))).astype(np.float32)
        flat[600:800] = dm
        flat[800:1000] = np.nextafter(dm, np.float32(np.inf))
        flat[1000:1200] = np.nextafter(dm, np.float32(0))
        flat[1200:1204] = [dmin, dmax, np.float32(dmin) * 0.999, np.float32(dmax) * 1.001]
        valid = rng.random((h, w)) > 0.1
        valid.reshape(-1)[1200:1204] = True
        vals[~valid] = np.where(rng.random((~valid).sum()) < 0.5, 0.0, np.nan).astype(np.float32)
        q = quantize_depth(DepthMap(np.where(valid, vals, 1.0), valid, intr), dmin, dmax, L)
        out[f"q{i}_vals"], out[f"q{i}_valid"], out[f"q{i}_codes"] = vals, valid, q.codes
        out[f"q{i}_param"] = np.array([dmin, dmax, L], dtype=np.float64)
        dq = dequantize_depth(q)
        out[f"q{i}_deq"] = dq.values
    out["nq"] = np.array(len(qcases))
    rcases = [(255, 1, 5), (255, 2, 8), (255, 3, 9), (255, 4, 7), (511, 5, 6), (255, 7, 8), (65535, 2, 9),
              (31, 3, 5), (255, 16, 8)]
    for i, (L, f, bits) in enumerate(rcases):
        h, w = int(rng.integers(20, 70)), int(rng.integers(20, 70))
        codes = rng.integers(1, L + 1, size=(h, w))
        codes[rng.random((h, w)) < 0.45] = 0
        codes[:f, :f] = 0                        # an all-invalid block
        q = QuantizedDepthMap(codes, levels=L, intrinsics=intr)
        ds = _downsample_codes_nearest_valid(q.codes, f)
        rq = _requantize_codes(QuantizedDepthMap(ds, q.d_min, q.d_max, q.levels, q.intrinsics), 2**bits - 1)
        out[f"r{i}_codes"], out[f"r{i}_param"] = q.codes, np.array([L, f, bits])
        out[f"r{i}_down"], out[f"r{i}_out"] = ds, rq.codes
    out["nr"] = np.array(len(rcases))
    np.savez_compressed(OUT / "mapstore.npz", **out)


def depthbuild_vectors():
    """Reference build_depth_map (depthbuild.py:249-375) on synth scenes: exact, noisy, outlier-corrupted,
    f32 fields, many views (V=20, 40); triangulate_pixel / depth_hypothesis on the noisy scene."""
    from types import SimpleNamespace
    from visloc.depthbuild import Observation, TriangulationConfig, build_depth_map, depth_hypothesis, \
        triangulate_pixel
    from visloc.synth import NoiseSpec, SceneSpec, corrupt, make_scene, oracle_field
    out = {}
    cases = [  # (n_cams, seed, spread, grid, sigma, outlier, f32, cfg kwargs)
        (6, 11, 0.25, 50, 0.0, 0.0, False, {}),
        (9, 13, 0.45, 40, 0.0, 0.4, False, {}),
        (6, 11, 0.25, 16, 0.3, 0.2, False, {}),
        (6, 11, 0.25, 30, 0.5, 0.3, True, {}),
        (21, 5, 0.5, 24, 0.4, 0.3, False, {"min_inliers": 3}),
        (41, 6, 0.6, 20, 0.4, 0.3, True, {"angular_threshold_rad": math.radians(1.0)}),
        (7, 3, 0.3, 20, 1.0, 0.5, False, {"confidence_threshold": 0.5, "max_refine_iters": 3}),
    ]
    for ci, (nc, seed, spread, grid, sigma, outl, f32, kw) in enumerate(cases):
        intr = CameraIntrinsics(70.0, 70.0, 70.0, 70.0, 140, 140)
        scene = make_scene(SceneSpec(num_cameras=nc, width=140, height=140, camera_spread=spread,
                                     camera_backoff=0.25, rotation_jitter_deg=3.0, seed=seed, intrinsics=intr))
        entry = SimpleNamespace(id=scene.view_id(0), pose=scene.cameras[0][0], intrinsics=scene.cameras[0][1])
        covis = [SimpleNamespace(id=scene.view_id(i), pose=scene.cameras[i][0], intrinsics=scene.cameras[i][1])
                 for i in range(1, nc)]
        fields = []
        for i in range(1, nc):
            f = oracle_field(scene, 0, i, grid, grid)
            if sigma > 0 or outl > 0:
                f = corrupt(f, NoiseSpec(sigma_px=sigma, outlier_fraction=outl), 100 * ci + i)
            if f32:
                f.targets = f.targets.astype(np.float32)
                f.confidence = f.confidence.astype(np.float32)
            fields.append(f)
        # a few cells with confidence on the gate boundary
        fields[0].confidence[0, :3] = [0.05, np.nextafter(0.05, 0), 0.0]
        cfg = TriangulationConfig(**kw)
        dm = build_depth_map(entry, covis, fields, cfg)
        p = f"c{ci}_"
        out[p + "targets"] = np.stack([f.targets for f in fields])
        out[p + "conf"] = np.stack([f.confidence for f in fields])
        out[p + "scale"] = np.array([fields[0].scale_x, fields[0].scale_y])
        out[p + "q"] = np.stack([entry.pose.q] + [c.pose.q for c in covis])
        out[p + "t"] = np.stack([entry.pose.t] + [c.pose.t for c in covis])
        out[p + "R"] = np.stack([entry.pose.R] + [c.pose.R for c in covis])
        out[p + "C"] = np.stack([entry.pose.center()] + [c.pose.center() for c in covis])
        out[p + "intr"] = np.array([[c.intrinsics.fx, c.intrinsics.fy, c.intrinsics.cx, c.intrinsics.cy,
                                     c.intrinsics.width, c.intrinsics.height] for c in [entry] + covis])
        out[p + "cfg"] = np.array([cfg.angular_threshold_rad, cfg.min_inliers, cfg.confidence_threshold,
                                   cfg.max_refine_iters, cfg.refine_tol])
        out[p + "depth"], out[p + "valid"] = dm.values, dm.valid
        if ci == 2:  # scalar path on every cell
            sx, sy = entry.intrinsics.width / grid, entry.intrinsics.height / grid
            sd, sn, hyp = [], [], []
            for row in range(grid):
                for col in range(grid):
                    obs = []
                    for i, f in enumerate(fields):
                        cc = float(f.confidence[row, col])
                        if cc >= cfg.confidence_threshold and cc > 0:
                            obs.append(Observation(covis[i].pose, covis[i].intrinsics, f.targets[row, col], cc))
                    px = np.array([(col + 0.5) * sx, (row + 0.5) * sy])
                    k = np.array([(px[0] - entry.intrinsics.cx) / entry.intrinsics.fx,
                                  (px[1] - entry.intrinsics.cy) / entry.intrinsics.fy, 1.0])
                    ray = entry.pose.R.T @ (k / np.linalg.norm(k))
                    r = triangulate_pixel(ray, entry.pose.center(), obs, cfg)
                    sd.append(np.nan if r is None else r[0])
                    sn.append(0 if r is None else r[1])
                    hyp.append([np.nan if (h := depth_hypothesis(ray, entry.pose.center(), o)) is None else h
                                for o in obs] + [np.inf] * (len(fields) - len(obs)))
            out[p + "scalar_depth"], out[p + "scalar_count"] = np.array(sd), np.array(sn)
            out[p + "scalar_hyp"] = np.array(hyp)
    out["n"] = np.array(len(cases))
    np.savez_compressed(OUT / "depthbuild.npz", **out)


class _LOCounter:
    """Counts the reference's LO calls: refine_pose with a TruncatedLoss inside
    ransac_pnp (posest.py:261-264; the final stage uses a CauchyLoss)."""

    def __enter__(self):
        import visloc.posest as P
        self.P, self.orig, self.n = P, P.refine_pose, 0

        def wrapped(*a, **k):
            loss = a[4] if len(a) > 4 else k.get("loss")
            if isinstance(loss, TruncatedLoss):
                self.n += 1
            return self.orig(*a, **k)

        P.refine_pose = wrapped
        return self

    def __exit__(self, *exc):
        self.P.refine_pose = self.orig


def _est_record(out, p, e, lo_calls):
    out[p + "q"], out[p + "t"] = e.pose.q, e.pose.t
    out[p + "flags"] = np.packbits(e.inlier_flags)
    out[p + "n"] = np.array(e.inlier_flags.size)
    out[p + "score"] = np.array(e.score)
    out[p + "iters"] = np.array(e.iterations)
    out[p + "conv"] = np.array(e.converged)
    out[p + "count"] = np.array(e.inlier_count)
    out[p + "lo_calls"] = np.array(lo_calls)


def baseline_vectors():
    """Reference ransac_pnp at the BASELINE single-query shapes:
    C1 (n=2k, eps=0.3, 10k fixed samples) and C4 (n=10k, eps=0.05, 100k fixed
    samples and the adaptive default), with the reference's LO-call counts."""
    cases = [
        # (name, n, outlier_frac, sigma, data seed, ransac seed, max_iterations, eta)
        ("c1", 2000, 0.7, 1.0, 41, 1, 10_000, 1e-300),
        ("c4", 10_000, 0.95, 1.0, 42, 2, 100_000, 1e-300),
        ("c4a", 10_000, 0.95, 1.0, 43, 3, 100_000, 1e-4),
    ]
    out = {"names": np.array([c[0] for c in cases]),
           "cases": np.array([c[1:] for c in cases], dtype=np.float64)}
    for name, n, of, sg, ds, rs, mi, eta in cases:
        px, X, w, _ = matches_a(n, of, sg, seed=ds)
        with _LOCounter() as lc:
            e = ransac_pnp((px, X, w), INTR_A, RansacConfig(seed=rs, max_iterations=mi, miss_probability=eta))
        _est_record(out, name + "_", e, lc.n)
        print(name, e.iterations, lc.n, e.inlier_count, e.converged, flush=True)
    np.savez_compressed(OUT / "baseline.npz", **out)


def _ref_scene(vmap, jobs, dcache):
    """Reference-typed copies of a generator-B scene (tests/synth_inputs.lifted_scene)."""
    from visloc.depthbuild import DepthMap
    from visloc.localizer import FieldPair, QueryJob
    from visloc.mapstore import QuantizedDepthMap
    from visloc.matchio import CorrespondenceField

    def intr(i):
        return CameraIntrinsics(i.fx, i.fy, i.cx, i.cy, i.width, i.height)

    class Entry:
        pass

    class Map:
        pass

    ents, depth = [], {}
    for e in vmap.entries:
        r = Entry()
        r.id, r.pose, r.intrinsics, r.descriptor = e.id, Pose(e.pose.q, e.pose.t), intr(e.intrinsics), e.descriptor
        r.qdepth = None
        if e.qdepth is not None:
            q = e.qdepth
            r.qdepth = QuantizedDepthMap(q.codes, q.d_min, q.d_max, q.levels, r.intrinsics)
        if dcache is not None and e.id in dcache:
            # the reference has no fp16 depth: its oracle is DepthMap(values=fp16.astype(f32))
            depth[e.id] = DepthMap(np.asarray(dcache[e.id].values).astype(np.float32), dcache[e.id].valid,
                                   r.intrinsics)
        ents.append(r)
    m = Map()
    m.entries = ents

    def cf(f):
        return CorrespondenceField(f.source_id, f.target_id, f.targets, f.confidence, f.scale_x, f.scale_y)

    rjobs = [QueryJob(j.query_id, intr(j.intrinsics), np.asarray(j.descriptor),
                      {k: FieldPair(cf(v.query_to_db), cf(v.db_to_query)) for k, v in j.fields.items()}, j.k_loc)
             for j in jobs]
    return m, rjobs, depth


def lift_full_vectors():
    """Reference lift + localize at the BASELINE lifted shapes on generator B
    (tests/synth_inputs.lifted_scene, f32 fields as a file-backed IMLC field):
    C5 (K=10, 117^2 fields, u8 log codes, and the fp16-depth variant, default
    config) and C2 (K=20, 83^2, f32 depth, 10k fixed samples).  Per (query,
    entry): the match count, sha256 of the pixel and weight bytes (bit-exact),
    every 61st world point and the per-coordinate sum of X; per query the
    localize estimate and the reference's LO-call count."""
    import hashlib
    from visloc.localizer import lift, localize
    from visloc.mapstore import dequantize_depth
    from synth_inputs import lifted_scene

    cases = [  # (name, K, g, depth, seed0, queries, max_iterations, eta)
        ("c5u8", 10, 117, "u8", 77, (0, 1), 100_000, 1e-4),
        ("c5f16", 10, 117, "f16", 77, (0, 1), 100_000, 1e-4),
        ("c2", 20, 83, "f32", 78, (0,), 10_000, 1e-300),
    ]
    out = {"names": np.array([c[0] for c in cases])}
    for name, K, g, dk, seed0, qs, mi, eta in cases:
        vmap, jobs, dc = lifted_scene(K, 0, g, seed=seed0, depth_kind=dk, fields="f32", only=list(qs))
        rmap, rjobs, rdepth = _ref_scene(vmap, jobs, dc)
        out[name + "_meta"] = np.array([K, g, seed0, mi], dtype=np.float64)
        out[name + "_eta"] = np.array(eta)
        out[name + "_queries"] = np.array(qs)
        for qi, rj in zip(qs, rjobs):
            p = f"{name}_q{qi}_"
            cnt, hpx, hw, xs, xsum = [], [], [], [], []
            for e in sorted(rmap.entries, key=lambda e: e.id):
                d = rdepth[e.id] if e.id in rdepth else dequantize_depth(e.qdepth)
                ms = lift(rj, e, d, 0.05)
                px = np.array([m.query_px for m in ms], dtype=np.float64).reshape(-1, 2)
                X = np.array([m.world_point for m in ms], dtype=np.float64).reshape(-1, 3)
                w = np.array([m.weight for m in ms], dtype=np.float64)
                cnt.append(len(ms))
                hpx.append(hashlib.sha256(np.ascontiguousarray(px).tobytes()).hexdigest())
                hw.append(hashlib.sha256(np.ascontiguousarray(w).tobytes()).hexdigest())
                xs.append(X[::61])
                xsum.append(X.sum(axis=0))
            out[p + "count"], out[p + "hpx"], out[p + "hw"] = np.array(cnt), np.array(hpx), np.array(hw)
            out[p + "Xs"], out[p + "Xsum"] = np.concatenate(xs), np.array(xsum)
            seed = 1_000_003 * seed0 + qi  # bench.query_seed
            with _LOCounter() as lc:
                est = localize(rj, rmap, RansacConfig(seed=seed, max_iterations=mi, miss_probability=eta),
                               depth_cache=dict(rdepth))
            _est_record(out, p + "loc_", est, lc.n)
            print(name, qi, sum(cnt), est.iterations, lc.n, est.inlier_count, est.converged, flush=True)
    np.savez_compressed(OUT / "lift_full.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate selected fixtures only, e.g. `make_golden.py mapstore`
        for name in sys.argv[1:]:
            globals()[f"{name}_vectors"]()
        sys.exit(0)
    depthbuild_vectors()
    mapstore_vectors()
    retrieval_vectors()
    imlc_vectors()
    lift_vectors()
    rng_vectors()
    R, t, px, X, w = p3p_vectors()
    score_vectors(R, t, px, X, w)
    msac_vectors()
    refine_vectors()
    ransac_vectors()
    baseline_vectors()
    lift_full_vectors()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
