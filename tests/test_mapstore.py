"""Depth-map codecs: oracle pinned to the reference's goldens,
the host threshold table checked exhaustively, GPU kernels bit-exact.

Reference: mapstore.py:96-134 (quantize / dequantize), :390-425 (nearest-valid
downsample, requantize), :428-497 (reduce_map); ports of
test_mapstore.py:46-108 and :207-280.
"""

import math

import numpy as np
import pytest

from oracle import mapstore as om


def _intr(w, h):
    from paper_2601_04185_b200.geometry import CameraIntrinsics
    return CameraIntrinsics(10.0, 10.0, w / 2, h / 2, w, h)


def _depth_map(values, valid=None):
    from paper_2601_04185_b200.mapstore import DepthMap
    values = np.asarray(values, dtype=np.float32)
    valid = np.ones_like(values, dtype=bool) if valid is None else valid
    h, w = values.shape
    return DepthMap(values=np.where(valid, values, 0).astype(np.float32), valid=valid, intrinsics=_intr(w, h))


# ----------------------------------------------------------------------------- CPU: oracle + host table
def test_oracle_matches_reference_goldens(golden):
    g = golden("mapstore")
    for i in range(int(g["nq"])):
        dmin, dmax, L = g[f"q{i}_param"]
        codes = om.quantize(g[f"q{i}_vals"], g[f"q{i}_valid"], dmin, dmax, int(L))
        np.testing.assert_array_equal(codes, g[f"q{i}_codes"])
        assert codes.dtype == g[f"q{i}_codes"].dtype
    for i in range(int(g["nr"])):
        L, f, bits = (int(x) for x in g[f"r{i}_param"])
        ds = om.downsample_nearest_valid(g[f"r{i}_codes"], f)
        np.testing.assert_array_equal(ds, g[f"r{i}_down"])
        rq = om.requantize(ds, L, 2 ** bits - 1)
        np.testing.assert_array_equal(rq, g[f"r{i}_out"])
        assert rq.dtype == g[f"r{i}_out"].dtype


def _codes_by_table(vals, valid, dmin, dmax, L):
    """What vl_quantize_depth computes: 1 + #{thresholds <= value} (as f32 bit patterns)."""
    from paper_2601_04185_b200.mapstore import quantize_thresholds
    thr = quantize_thresholds(float(dmin), float(dmax), int(L)).view(np.uint32)
    bits = np.asarray(vals, dtype=np.float32).view(np.uint32)
    c = 1 + np.searchsorted(thr, bits, side="right")
    return np.where(valid, c, 0)


def test_threshold_table_reproduces_goldens(golden):
    g = golden("mapstore")
    for i in range(int(g["nq"])):
        dmin, dmax, L = g[f"q{i}_param"]
        v = np.where(g[f"q{i}_valid"], g[f"q{i}_vals"], 1.0).astype(np.float32)
        np.testing.assert_array_equal(_codes_by_table(v, g[f"q{i}_valid"], dmin, dmax, L), g[f"q{i}_codes"])


def test_threshold_table_is_exact_for_every_f32_default_params():
    """Every f32 from below d_min to above d_max (default 0.25-128 m, 255 levels)."""
    dmin, dmax, L = 0.25, 128.0, 255
    lo = int(np.float32(dmin * 0.5).view(np.uint32))
    hi = int(np.float32(dmax * 2.0).view(np.uint32))
    from paper_2601_04185_b200.mapstore import quantize_thresholds
    thr = quantize_thresholds(dmin, dmax, L).view(np.uint32)
    step = 1 << 23
    for a in range(lo, hi, step):
        bits = np.arange(a, min(a + step, hi), dtype=np.uint32)
        ref = om.quantize(bits.view(np.float32), np.ones(bits.size, bool), dmin, dmax, L).astype(np.int64)
        got = 1 + np.searchsorted(thr, bits, side="right")
        np.testing.assert_array_equal(got, ref)


def test_threshold_table_levels_edge_cases():
    from paper_2601_04185_b200.mapstore import quantize_thresholds
    assert quantize_thresholds(0.25, 128.0, 1).size == 0
    t = quantize_thresholds(0.25, 128.0, 2)
    assert t.size == 1 and om.quantize(np.array([t[0]]), [True], 0.25, 128.0, 2)[0] == 2
    assert om.quantize(np.array([np.nextafter(t[0], np.float32(0))]), [True], 0.25, 128.0, 2)[0] == 1
    t16 = quantize_thresholds(0.25, 128.0, 65535)
    assert t16.size == 65534 and np.all(np.diff(t16.view(np.uint32).astype(np.int64)) >= 0)


# ----------------------------------------------------------------------------- GPU
gpu = pytest.mark.gpu


@gpu
def test_gpu_quantize_goldens(golden):
    from paper_2601_04185_b200.mapstore import quantize_depth_batch
    g = golden("mapstore")
    for i in range(int(g["nq"])):
        dmin, dmax, L = g[f"q{i}_param"]
        valid = g[f"q{i}_valid"]
        dm = _depth_map(np.where(valid, g[f"q{i}_vals"], 1.0), valid)
        q, = quantize_depth_batch([dm], float(dmin), float(dmax), int(L))
        np.testing.assert_array_equal(q.codes, g[f"q{i}_codes"])
        assert q.codes.dtype == g[f"q{i}_codes"].dtype and q.levels == int(L)


@gpu
def test_gpu_quantize_batch_mixed_shapes_and_f16():
    from paper_2601_04185_b200.mapstore import DepthMap, quantize_depth_batch
    rng = np.random.default_rng(5)
    maps = []
    for k in range(70):  # > 64 maps: two launches
        h, w = int(rng.integers(1, 90)), int(rng.integers(1, 90))
        v = np.exp(rng.uniform(math.log(0.05), math.log(400), (h, w)))
        valid = rng.random((h, w)) > 0.2
        dt = np.float16 if k % 3 == 0 else np.float32
        maps.append(DepthMap(np.where(valid, v, 1.0).astype(dt), valid, _intr(w, h)))
    for L in (255, 2000):
        out = quantize_depth_batch(maps, 0.25, 128.0, L)
        for m, q in zip(maps, out):
            ref = om.quantize(np.asarray(m.values, dtype=np.float32), m.valid, 0.25, 128.0, L)
            np.testing.assert_array_equal(q.codes, ref)


@gpu
def test_gpu_quantize_every_f32_default_params():
    """Exhaustive: all f32 in [d_min/2, 2 d_max] through the kernel vs the reference formula."""
    from paper_2601_04185_b200.mapstore import DepthMap, quantize_depth
    lo = int(np.float32(0.125).view(np.uint32))
    hi = int(np.float32(256.0).view(np.uint32))
    bits = np.arange(lo, hi, dtype=np.uint32)
    n = bits.size
    w = 8192
    pad = (-n) % w
    vals = np.concatenate([bits, np.full(pad, bits[-1], np.uint32)]).view(np.float32).reshape(-1, w)
    q = quantize_depth(DepthMap(vals, np.ones(vals.shape, bool), _intr(w, vals.shape[0])))
    got = q.codes.reshape(-1)[:n]
    step = 1 << 23
    for a in range(0, n, step):
        ref = om.quantize(bits[a:a + step].view(np.float32), np.ones(min(step, n - a), bool), 0.25, 128.0, 255)
        np.testing.assert_array_equal(got[a:a + step], ref)


@gpu
def test_gpu_reduce_goldens(golden):
    from paper_2601_04185_b200.mapstore import QuantizedDepthMap, _reduce_codes_batch
    g = golden("mapstore")
    for i in range(int(g["nr"])):
        L, f, bits = (int(x) for x in g[f"r{i}_param"])
        q = QuantizedDepthMap(g[f"r{i}_codes"], levels=L)
        ds, = _reduce_codes_batch([q], f, L)                  # downsample only
        np.testing.assert_array_equal(ds, g[f"r{i}_down"])
        out, = _reduce_codes_batch([q], f, 2 ** bits - 1)      # fused downsample + requantize
        np.testing.assert_array_equal(out, g[f"r{i}_out"])
        assert out.dtype == g[f"r{i}_out"].dtype


# ---- ports of the reference's unit tests (test_mapstore.py:46-108, :207-280) ----
@gpu
def test_gpu_reference_quantization_kats():
    from paper_2601_04185_b200.mapstore import QuantizedDepthMap, dequantize_depth, quantize_depth
    np.testing.assert_array_equal(quantize_depth(_depth_map([[0.25, 128.0]])).codes, [[1, 255]])
    assert quantize_depth(_depth_map([[0.25 * math.sqrt(512.0)]])).codes[0, 0] == 128
    np.testing.assert_array_equal(quantize_depth(_depth_map([[0.01, 500.0]])).codes, [[1, 255]])
    q = quantize_depth(_depth_map([[1.0, 2.0]], valid=np.array([[True, False]])))
    assert q.codes[0, 0] > 0 and q.codes[0, 1] == 0
    codes = np.arange(0, 256, dtype=np.uint8).reshape(16, 16)
    q0 = QuantizedDepthMap(codes.copy())
    np.testing.assert_array_equal(quantize_depth(dequantize_depth(q0), q0.d_min, q0.d_max, q0.levels).codes, codes)
    rng = np.random.default_rng(0)
    d = np.exp(rng.uniform(math.log(0.25), math.log(128.0), 200_000)).astype(np.float32)
    side = int(math.sqrt(d.size))
    dm = _depth_map(d[: side * side].reshape(side, side))
    back = dequantize_depth(quantize_depth(dm))
    rel = np.abs(back.values.astype(np.float64) - dm.values.astype(np.float64)) / dm.values.astype(np.float64)
    assert rel.max() <= math.expm1(math.log(512.0) / (2 * 254)) * (1 + 1e-6)
    d = np.linspace(0.25, 128.0, 4096, dtype=np.float32).reshape(64, 64)
    assert np.all(np.diff(quantize_depth(_depth_map(d)).codes.reshape(-1).astype(np.int32)) >= 0)
    d = np.exp(np.random.default_rng(1).uniform(math.log(0.25), math.log(128.0), 10_000))
    dm = _depth_map(d.reshape(100, 100).astype(np.float32))
    back = dequantize_depth(quantize_depth(dm, levels=127))
    rel = np.abs(back.values.astype(np.float64) - dm.values.astype(np.float64)) / dm.values.astype(np.float64)
    assert rel.max() <= math.expm1(math.log(512.0) / (2 * 126)) * (1 + 1e-6)
    with pytest.raises(ValueError):
        quantize_depth(_depth_map([[1.0]]), d_min=2.0, d_max=1.0)


def _entries(n=3, size=24):
    import io
    from PIL import Image
    from paper_2601_04185_b200.geometry import Pose
    from paper_2601_04185_b200.mapstore import MapEntry, QuantizedDepthMap
    rng = np.random.default_rng(2)
    out = []
    for i in range(n):
        buf = io.BytesIO()
        Image.fromarray(rng.integers(0, 255, (size, size, 3), dtype=np.uint8), mode="RGB").save(buf, format="PNG")
        codes = rng.integers(0, 256, (size // 2, size // 2)).astype(np.uint8)
        out.append(MapEntry(id=f"im{i:02d}", pose=Pose.identity(), intrinsics=_intr(size, size),
                            rgb_payload=buf.getvalue(), rgb_codec="png",
                            qdepth=QuantizedDepthMap(codes, intrinsics=_intr(size, size)),
                            descriptor=rng.normal(size=8)))
    return out


@gpu
def test_gpu_reference_reduce_map_ports():
    import io
    from PIL import Image
    from paper_2601_04185_b200.mapstore import Map, MapEntry, QuantizedDepthMap, reduce_map
    vmap = Map(entries=_entries())
    r = reduce_map(vmap, 1, 1.0, 90, 1, 8)
    for a, b in zip(vmap.entries, r.entries):
        assert np.array_equal(a.qdepth.codes, b.qdepth.codes) and a.rgb_payload == b.rgb_payload
        assert np.array_equal(a.descriptor, b.descriptor)
    base = vmap.entries[0]
    many = [MapEntry(id=f"im{i:02d}", pose=base.pose, intrinsics=base.intrinsics, rgb_payload=base.rgb_payload,
                     rgb_codec="png", qdepth=base.qdepth, descriptor=base.descriptor) for i in range(16)]
    assert [e.id for e in reduce_map(Map(entries=many), keyframe_stride=8).entries] == ["im00", "im08"]
    for e in reduce_map(vmap, 1, 1.0, 90, 1, 7).entries:
        assert e.qdepth.levels == 127 and e.qdepth.codes.max() <= 127
        np.testing.assert_array_equal(e.qdepth.codes, om.requantize(vmap.entry(e.id).qdepth.codes, 255, 127))
    r9 = reduce_map(vmap, 1, 1.0, 90, 1, 9)
    assert r9.entries[0].qdepth.codes.dtype == np.uint16 and r9.entries[0].qdepth.levels == 511
    codes = np.zeros((4, 4), dtype=np.uint8)
    codes[0, 0], codes[1, 1], codes[2, 3] = 10, 20, 30
    base.qdepth = QuantizedDepthMap(codes)
    out = reduce_map(Map(entries=[base]), 1, 1.0, 90, 2, 8).entries[0].qdepth.codes
    assert out.shape == (2, 2) and out[0, 0] == 10 and out[0, 1] == 0 and out[1, 1] == 30
    codes = np.zeros((3, 3), dtype=np.uint8)
    codes[0, 0], codes[1, 1] = 10, 20
    base.qdepth = QuantizedDepthMap(codes)
    out = reduce_map(Map(entries=[base]), 1, 1.0, 90, 3, 8).entries[0].qdepth.codes
    assert out.shape == (1, 1) and out[0, 0] == 20
    with pytest.raises(ValueError):  # RGB re-encoding: map storage, out of scope
        reduce_map(Map(entries=_entries(1)), 1, 2.0, 90, 1, 8)
    with pytest.raises(ValueError):
        reduce_map(vmap, 0)
    with pytest.raises(ValueError):
        reduce_map(vmap, 1, 1.0, 90, 1, 12)
