"""IMLC field ingestion against the reference's read_field.

Golden blobs and verdicts come from the real reference (tests/golden/imlc.npz,
``make_golden.imlc_vectors``): valid fields (NaN targets at confidence 0),
every truncation point, bad magic/version, trailing bytes, zero/huge grids
and each record-content rule.  CPU tests cover the C header parser
(``vl_imlc_parse``) and the host ``read_field``; GPU tests cover the in-place
record lift and the GPU content validation.
"""

import json

import numpy as np
import pytest


def _cases(golden):
    d = golden("imlc")
    return [(d[f"blob{i}"].tobytes(), json.loads(str(d[f"expect{i}"])), d, i) for i in range(int(d["n"]))]


CONTENT = {"conf_gt1", "conf_neg", "conf_nan", "target_nan", "target_inf"}


def _check_exc(exc, exp):
    assert type(exc).__name__ == exp["cls"], (exp["name"], type(exc).__name__)
    assert str(exc) == exp["msg"], exp["name"]
    assert exc.offset == exp["offset"], exp["name"]


def test_header_parse_matches_reference(golden):
    from paper_2601_04185_b200 import matchio
    for blob, exp, _, _ in _cases(golden):
        if exp["name"] in CONTENT:
            info = matchio.parse_header(blob)  # framing is fine; content is checked by the lift
            assert info.grid_w * info.grid_h * 12 + info.records_off == len(blob)
            continue
        if exp["ok"]:
            info = matchio.parse_header(blob)
            for k in ("source_id", "target_id", "grid_w", "grid_h", "scale_x", "scale_y"):
                assert getattr(info, k) == exp[k], k
            continue
        with pytest.raises(matchio.FieldFormatError) as ei:
            matchio.parse_header(blob)
        _check_exc(ei.value, exp)


def test_read_field_matches_reference(golden, tmp_path):
    from paper_2601_04185_b200 import matchio
    for blob, exp, d, i in _cases(golden):
        p = tmp_path / f"{i}.imlc"
        p.write_bytes(blob)
        if exp["ok"]:
            f = matchio.read_field(p)
            assert f.targets.dtype == np.float32 and f.confidence.dtype == np.float32
            # byte-exact, NaN payloads included
            assert f.targets.tobytes() == d[f"targets{i}"].tobytes()
            assert f.confidence.tobytes() == d[f"conf{i}"].tobytes()
            assert (f.source_id, f.target_id, f.scale_x, f.scale_y) == (
                exp["source_id"], exp["target_id"], exp["scale_x"], exp["scale_y"])
            # write -> read round trip is bit-exact (matchio.write_field contract)
            q = tmp_path / f"{i}_rt.imlc"
            matchio.write_field(f, q)
            assert q.read_bytes() == blob
        else:
            with pytest.raises(matchio.FieldFormatError) as ei:
                matchio.read_field(p)
            _check_exc(ei.value, exp)


def test_parse_rejects_null():
    import ctypes as C
    from paper_2601_04185_b200 import _lib
    h = _lib.ImlcHeader()
    assert _lib.lib().vl_imlc_parse(None, 5, C.byref(h)) == _lib.VL_ERR_INVALID
    assert _lib.lib().vl_imlc_parse(None, 0, None) == _lib.VL_ERR_INVALID


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_gpu_gate_from_arena_matches_reference(golden):
    """filter_matches_arrays on in-place IMLC records == the planar path == reference gate."""
    from paper_2601_04185_b200 import matchio
    blob, exp, d, i = _cases(golden)[0]
    assert exp["ok"]
    arena = matchio.FieldArena([blob, blob])  # two copies: exercises alignment padding
    assert all(f.records_offset % 16 == 0 for f in arena.fields)
    tg, cf = d[f"targets{i}"], d[f"conf{i}"]
    for thr in (0.0, 0.05, 0.5, 1.0):
        src, tgt, conf, cell = matchio.filter_matches_arrays(arena[1], thr)
        mask = (cf >= np.float32(thr)) & (cf > 0)
        rows, cols = np.nonzero(mask)
        ref_src = np.stack([(cols + 0.5) * exp["scale_x"], (rows + 0.5) * exp["scale_y"]], -1)
        assert np.array_equal(src, ref_src)
        assert np.array_equal(tgt, tg[rows, cols].astype(np.float64))
        assert np.array_equal(conf, cf[rows, cols].astype(np.float64))
        assert np.array_equal(cell, rows * exp["grid_w"] + cols)
        planar = matchio.CorrespondenceField("a", "b", tg, cf, exp["scale_x"], exp["scale_y"])
        p2 = matchio.filter_matches_arrays(planar, thr)
        for a, b in zip((src, tgt, conf, cell), p2):
            assert np.array_equal(a, b)


@pytest.mark.gpu
def test_gpu_content_validation_matches_reference(golden):
    from paper_2601_04185_b200 import matchio
    for blob, exp, _, _ in _cases(golden):
        if exp["name"] not in CONTENT:
            continue
        arena = matchio.FieldArena([blob])
        with pytest.raises(matchio.FieldFormatError) as ei:
            matchio.filter_matches_arrays(arena[0], 0.05)
        _check_exc(ei.value, exp)


@pytest.mark.gpu
def test_gpu_lift_from_imlc_equals_reference(golden):
    """Reference lift goldens (f32 fields) reproduced from IMLC blobs read in place."""
    from paper_2601_04185_b200 import localizer as L
    from paper_2601_04185_b200 import matchio
    from scene_io import unpack_scene
    d = golden("lift")
    vmap, jobs = unpack_scene(d)
    entries = vmap.entries
    n = int(d["nlift"])
    checked = 0
    for k in range(n):
        j, ei, dk, fdt = (int(v) for v in d[f"L{k}_meta"])
        if fdt != 1:
            continue
        job, e = jobs[j], entries[ei]
        fp = job.fields[e.id]
        blobs = [matchio.field_bytes(matchio.CorrespondenceField(
            f.source_id, f.target_id, np.asarray(f.targets, np.float32), np.asarray(f.confidence, np.float32),
            f.scale_x, f.scale_y)) for f in (fp.query_to_db, fp.db_to_query)]
        arena = matchio.FieldArena(blobs)
        job2 = L.QueryJob(job.query_id, job.intrinsics, job.descriptor,
                          {e.id: L.FieldPair(arena[0], arena[1])}, job.k_loc)
        if dk == 0:
            depth = L.DepthMap(d[f"gt{ei}_values"], d[f"gt{ei}_valid"], e.intrinsics)
        else:
            depth = L.dequantize_depth(e.qdepth)
        px, X, w = L.lift_arrays(job2, e, depth, 0.05)
        assert np.array_equal(px.cpu().numpy(), d[f"L{k}_px"])
        Xg = X.cpu().numpy()
        assert Xg.shape == d[f"L{k}_X"].shape
        assert np.abs(Xg - d[f"L{k}_X"]).max(initial=0.0) < 1e-13  # reference dgemm order (test_lift.py)
        assert np.array_equal(w.cpu().numpy(), d[f"L{k}_w"])
        checked += 1
    assert checked >= 3


@pytest.mark.gpu
def test_gpu_localize_pipelined_equals_batch(golden):
    """Micro-batched serving loop (per-batch arenas, side-stream uploads) == one localize_batch."""
    from paper_2601_04185_b200 import localizer as L
    from paper_2601_04185_b200 import matchio
    from paper_2601_04185_b200.posest import RansacConfig
    from scene_io import unpack_scene
    vmap, jobs = unpack_scene(golden("lift"))
    cfg = RansacConfig(seed=3)
    seeds = [40 + j for j in range(len(jobs))]
    batches = []
    for lo, hi in ((0, 1), (1, 3), (3, len(jobs))):
        blobs, keys = [], []
        for j in range(lo, hi):
            for eid, fp in sorted(jobs[j].fields.items()):
                for f in (fp.query_to_db, fp.db_to_query):
                    blobs.append(matchio.field_bytes(matchio.CorrespondenceField(
                        f.source_id, f.target_id, np.asarray(f.targets, np.float32),
                        np.asarray(f.confidence, np.float32), f.scale_x, f.scale_y)))
                keys.append((j, eid))
        arena = matchio.FieldArena(blobs)
        bj = []
        for j in range(lo, hi):
            fields = {eid: L.FieldPair(arena[2 * k], arena[2 * k + 1]) for k, (jj, eid) in enumerate(keys) if jj == j}
            bj.append(L.QueryJob(jobs[j].query_id, jobs[j].intrinsics, jobs[j].descriptor, fields, jobs[j].k_loc))
        batches.append((bj, arena))
    flat = [j for b, _ in batches for j in b]
    ref = L.localize_batch(flat, vmap, cfg, seeds=seeds, depth_cache={})
    import torch
    for lanes, nbuf in ((1, 1), (2, 2), (2, 3), (3, 1)):
        bufs = [torch.empty(max(a.host.numel() for _, a in batches), dtype=torch.uint8, device="cuda")
                for _ in range(nbuf)]
        got = L.localize_pipelined(batches, vmap, cfg, seeds=seeds, depth_cache={}, buffers=bufs, lanes=lanes)
        assert len(got) == len(ref)
        for a, b in zip(ref, got):
            assert np.array_equal(a.pose.q, b.pose.q) and np.array_equal(a.inlier_flags, b.inlier_flags)
            assert a.iterations == b.iterations and a.score == b.score
    # an error in one lane's batch surfaces on the caller (no lane left waiting)
    bad = [(list(b), a) for b, a in batches]
    j0 = bad[1][0][0]
    bad[1][0][0] = L.QueryJob(j0.query_id, L.CameraIntrinsics(1.0, 1.0, 0.0, 0.0, 7, 7), j0.descriptor,
                              j0.fields, j0.k_loc)
    with pytest.raises(ValueError, match="does not span image 7x7"):
        L.localize_pipelined(bad, vmap, cfg, seeds=seeds, depth_cache={}, lanes=2)
