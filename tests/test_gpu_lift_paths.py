"""Every code path of the lift kernels against the oracle lift (localizer.py:134-197).

The kernels pick block-uniform paths: IMLC records staged by one bulk copy
(16-B aligned payloads) or read per cell (4-B aligned payloads, planar
fields); db->query taps and ray quotients from per-column / per-row tables
(grid width <= 512 and a block spanning <= 72 rows) or computed per cell;
one template per depth kind (f32, f16, u8 / u16 codes).  Each combination
must give the oracle's matches in the reference order: pixels and weights
bit-exact, world points within 1e-12.
"""

import numpy as np
import pytest

from oracle import geometry as og
from oracle import lift as ol

pytestmark = pytest.mark.gpu

THR = 0.05


@pytest.fixture(scope="module")
def vl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_04185_b200.localizer as L
    return L


def _scene(gw, gh, kind, seed):
    """One database entry (W x H image, depth at grid resolution gw x gh) and a
    query with bidirectional f32 fields on the same grid."""
    from paper_2601_04185_b200.geometry import CameraIntrinsics, Pose, rotvec_to_quat
    rng = np.random.default_rng(seed)
    W, H = 4.0 * gw, 4.0 * gh
    intr = CameraIntrinsics(0.8 * W, 0.8 * W, W / 2, H / 2, int(W), int(H))
    pose = Pose(rotvec_to_quat(rng.normal(size=3) * 0.1), rng.normal(size=3))
    depth = rng.uniform(1.0, 9.0, (gh, gw)).astype(np.float32)
    valid = rng.random((gh, gw)) > 0.1
    depth[~valid] = 0.0

    def field():
        tg = np.stack([rng.uniform(-2, W + 2, (gh, gw)), rng.uniform(-2, H + 2, (gh, gw))], -1).astype(np.float32)
        cf = rng.uniform(0, 1, (gh, gw)).astype(np.float32)
        cf[rng.random((gh, gw)) < 0.2] = 0.0
        return tg, cf

    return intr, pose, depth, valid, field(), field()


def _depth_obj(vl, kind, depth, valid, intr):
    if kind == "u8":
        span = np.log(128.0) - np.log(0.25)
        uq = (np.log(np.clip(depth.astype(np.float64), 0.25, 128.0)) - np.log(0.25)) / span
        codes = np.where(valid, 1 + np.floor(uq * 254 + 0.5), 0).astype(np.uint8)
        q = vl.QuantizedDepthMap(codes, 0.25, 128.0, 255, intr)
        vals, ok = ol.dequantize(codes, 0.25, 128.0, 255)
        return q, vals, ok
    if kind == "u16":
        span = np.log(128.0) - np.log(0.25)
        uq = (np.log(np.clip(depth.astype(np.float64), 0.25, 128.0)) - np.log(0.25)) / span
        codes = np.where(valid, 1 + np.floor(uq * 1022 + 0.5), 0).astype(np.uint16)
        q = vl.QuantizedDepthMap(codes, 0.25, 128.0, 1023, intr)
        vals, ok = ol.dequantize(codes, 0.25, 128.0, 1023)
        return q, vals, ok
    dt = np.float16 if kind == "f16" else np.float32
    d = vl.DepthMap(depth.astype(dt), valid, intr)
    return d, np.asarray(d.values).astype(np.float32), valid


def _oracle(intr, pose, vals, ok, f_db2q, f_q2db):
    I = intr
    return ol.lift((f_db2q[0], f_db2q[1], 4.0, 4.0), (f_q2db[0], f_q2db[1], 4.0, 4.0), vals, ok,
                   (I.fx, I.fy, I.cx, I.cy), (I.width, I.height), og.q2R(pose.q), pose.t, THR)


def _check(got, ref):
    px, X, w = (a.cpu().numpy() if hasattr(a, "cpu") else a for a in got)
    assert px.shape == ref[0].shape
    assert np.array_equal(px, ref[0]) and np.array_equal(w, ref[2])
    assert np.abs(X - ref[1]).max(initial=0.0) <= 1e-12


# (117, 117): column/row tables; (600, 7): grid wider than the tables;
# (20, 300): a block spans > 72 rows; (3, 5): a 15-cell segment
@pytest.mark.parametrize("gw,gh", [(117, 117), (600, 7), (20, 300), (3, 5)])
@pytest.mark.parametrize("kind", ["f32", "f16", "u8", "u16"])
def test_lift_paths_vs_oracle(vl, gw, gh, kind):
    from paper_2601_04185_b200.localizer import FieldPair, QueryJob
    intr, pose, depth, valid, f1, f2 = _scene(gw, gh, kind, seed=gw * 7 + gh)

    class Entry:
        pass

    e = Entry()
    e.id, e.pose, e.intrinsics = "db", pose, intr
    dobj, vals, ok = _depth_obj(vl, kind, depth, valid, intr)
    ref = _oracle(intr, pose, vals, ok, f1, f2)
    job = QueryJob("q", intr, np.zeros(4), {"db": FieldPair(
        vl.CorrespondenceField("q", "db", f2[0], f2[1], 4.0, 4.0),
        vl.CorrespondenceField("db", "q", f1[0], f1[1], 4.0, 4.0))})
    _check(vl.lift_arrays(job, e, dobj, THR), ref)  # planar f32 fields


@pytest.mark.parametrize("gw,gh", [(117, 117), (600, 7), (20, 300), (3, 5)])
@pytest.mark.parametrize("kind", ["u8", "f32", "f16", "u16"])
def test_lift_imlc_aligned_and_unaligned_records(vl, gw, gh, kind):
    """IMLC records 16-B aligned (bulk-copy staging: the grouped count loop)
    and at a 4-B offset (per-cell loads), every depth kind."""
    import torch
    from paper_2601_04185_b200 import _lib
    from paper_2601_04185_b200.localizer import _depth_record, _call_lift, FieldPair, QueryJob
    from paper_2601_04185_b200.matchio import FieldArena, field_bytes
    intr, pose, depth, valid, f1, f2 = _scene(gw, gh, kind, seed=gw + gh)

    class Entry:
        pass

    e = Entry()
    e.id, e.pose, e.intrinsics = "db", pose, intr
    dobj, vals, ok = _depth_obj(vl, kind, depth, valid, intr)
    ref = _oracle(intr, pose, vals, ok, f1, f2)
    fq = vl.CorrespondenceField("q", "db", f2[0], f2[1], 4.0, 4.0)
    fd = vl.CorrespondenceField("db", "q", f1[0], f1[1], 4.0, 4.0)
    arena = FieldArena([field_bytes(fq), field_bytes(fd)])
    job = QueryJob("q", intr, np.zeros(4), {"db": FieldPair(arena[0], arena[1])})
    _check(vl.lift_arrays(job, e, dobj, THR), ref)  # arena: records 16-B aligned
    # the same records copied to a device buffer at a 4-B (not 16-B) aligned offset
    keep = {}
    rec = _depth_record(e, dobj, keep)
    cells = gw * gh
    recs = [np.concatenate([t.reshape(-1, 2), c.reshape(-1, 1)], 1).astype(np.float32) for t, c in (f1, f2)]
    buf = torch.zeros(2 * (3 * cells + 8) + 4, dtype=torch.float32, device="cuda")
    base = 1  # one float = 4 bytes past a 16-B aligned allocation
    off = [base, base + 3 * cells + 4]
    for o, r in zip(off, recs):
        buf[o:o + 3 * cells] = torch.from_numpy(r.reshape(-1)).cuda()
    table = np.zeros(2, dtype=_lib.LIFT_SEGMENT_DTYPE)
    for k, (direction, o) in enumerate([(0, off[0]), (1, off[1])]):
        table[k]["direction"], table[k]["grid_w"], table[k]["grid_h"] = direction, gw, gh
        table[k]["scale_x"], table[k]["scale_y"] = 4.0, 4.0
        table[k]["layout"] = _lib.LIFT_IMLC
        table[k]["targets"] = buf.data_ptr() + 4 * o
    assert (int(table[0]["targets"]) & 15) != 0
    cap = 2 * cells
    px = torch.empty((cap, 2), dtype=torch.float64, device="cuda")
    X = torch.empty((cap, 3), dtype=torch.float64, device="cuda")
    w = torch.empty((cap,), dtype=torch.float64, device="cuda")
    ent = torch.empty((cap,), dtype=torch.int32, device="cuda")
    offs = np.zeros(3, dtype=np.int64)
    flags = np.zeros(2, dtype=np.int32)
    deps = (_lib.LiftDepth * 1)(rec)
    _call_lift(table, 2, deps, 1, False, THR, 0, px, X, w, ent, cap, offs, flags, [fd, fq])
    n = int(offs[-1])
    _check((px[:n], X[:n], w[:n]), ref)


def test_lift_grouped_loops_equal_per_cell_loops(tmp_path):
    """The grouped count loop over staged IMLC records (default) and the
    per-cell loop (VISLOC_LIFT_GROUPED=0, read once per process) give the same
    matches bit for bit on a C5-shaped lift (u8 and f16 depth, both
    directions, 117 x 117 fields)."""
    import os
    import subprocess
    import sys
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = (
        "import sys, numpy as np\n"
        f"sys.path[:0] = [{root!r}, {os.path.join(root, 'tests')!r}]\n"
        "from synth_inputs import lifted_scene\n"
        "import paper_2601_04185_b200.localizer as L\n"
        "from paper_2601_04185_b200.matchio import FieldArena, field_bytes\n"
        "from paper_2601_04185_b200.localizer import FieldPair\n"
        "out = {}\n"
        "for kind in ('u8', 'f16'):\n"
        "    vmap, jobs, dc = lifted_scene(3, 2, 117, seed=5, depth_kind=kind, fields='f32')\n"
        "    for qi, job in enumerate(jobs):\n"
        "        for e in vmap.entries:\n"
        "            fp = job.fields[e.id]\n"
        "            ar = FieldArena([field_bytes(fp.query_to_db), field_bytes(fp.db_to_query)])\n"
        "            job.fields[e.id] = FieldPair(ar[0], ar[1])\n"
        "            d = e.qdepth if kind == 'u8' else dc[e.id]\n"
        "            px, X, w = (a.cpu().numpy() if hasattr(a, 'cpu') else np.asarray(a) for a in L.lift_arrays(job, e, d, 0.05))\n"
        "            for nm, a in (('px', px), ('X', X), ('w', w)):\n"
        "                out[f'{kind}_{qi}_{e.id}_{nm}'] = a\n"
        "np.savez(sys.argv[1], **out)\n")
    res = {}
    for v in ("0", "1"):
        f = tmp_path / f"lift_{v}.npz"
        env = dict(os.environ, VISLOC_LIFT_GROUPED=v)
        subprocess.run([sys.executable, "-c", script, str(f)], check=True, env=env, cwd=root)
        res[v] = np.load(f)
    assert len(res["0"].files) == len(res["1"].files) > 0
    for k in res["0"].files:
        assert np.array_equal(res["0"][k], res["1"][k]), k
    assert sum(res["0"][k].shape[0] for k in res["0"].files if k.endswith("_w")) > 10000
