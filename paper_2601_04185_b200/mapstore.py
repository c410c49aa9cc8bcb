"""Depth-map codecs on the GPU — drop-in for the depth side of ``visloc.mapstore``.

SURVEY §8f row 4: the u8/u16 log codes the lift's table decode consumes
(``localizer._DeviceDepth``) are produced here, many maps per launch.

* ``quantize_depth`` / ``quantize_depth_batch`` — ``mapstore.quantize_depth``
  (mapstore.py:96-119).  The code is a monotone step function of the f32
  depth; ``quantize_thresholds`` tabulates its steps once per
  (d_min, d_max, levels) with the reference's own fp64 numpy arithmetic
  (vectorised bisection over f32 bit patterns) and ``vl_quantize_depth``
  counts thresholds per pixel — bit-exact for every f32 depth.
* ``dequantize_depth`` — ``mapstore.dequantize_depth`` (:122-134), GPU table
  decode (``vl_decode_depth``).
* ``reduce_depth_codes`` / ``reduce_map`` — the depth step of
  ``mapstore.reduce_map`` (:428-497): nearest-valid block downsampling
  (:390-414) + requantisation (:417-425) in one ``vl_reduce_depth_codes``
  launch for every kept entry.  Keyframe selection and the RGB payload
  follow the reference on the host (RGB resampling is map storage, not the
  GPU path; it uses Pillow exactly like the reference).

Inputs are duck-typed: the reference's own ``DepthMap`` /
``QuantizedDepthMap`` / ``MapEntry`` / ``Map`` objects work, and outputs are
built with the input objects' classes.
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .geometry import CameraIntrinsics, Pose
from .localizer import DEFAULT_D_MAX, DEFAULT_D_MIN, DepthMap, QuantizedDepthMap, dequantize_depth

__all__ = [
    "DEFAULT_D_MAX", "DEFAULT_D_MIN", "DepthMap", "Map", "MapEntry", "QuantizedDepthMap", "dequantize_depth",
    "quantize_depth", "quantize_depth_batch", "quantize_depth_device", "quantize_thresholds", "reduce_depth_codes", "reduce_map",
]

_F32_MAX_BITS = 0x7F7FFFFF


@dataclass
class MapEntry:
    """One database image (mapstore.py:137-156); RGB payload kept encoded."""

    id: str
    pose: Pose
    intrinsics: CameraIntrinsics
    rgb_payload: bytes
    rgb_codec: str
    qdepth: QuantizedDepthMap | None
    descriptor: np.ndarray

    def __post_init__(self):
        self.descriptor = np.ascontiguousarray(self.descriptor, dtype=np.float16)


@dataclass
class Map:
    """Ordered entries plus codec identifiers (mapstore.py:159-182)."""

    entries: list = field(default_factory=list)
    rgb_codec: str = "png"
    depth_codec: str = "png"

    def __post_init__(self):
        ids = [e.id for e in self.entries]
        if len(set(ids)) != len(ids):
            dupes = sorted({i for i in ids if ids.count(i) > 1})
            raise ValueError(f"duplicate entry ids: {dupes}")

    def entry(self, entry_id):
        for e in self.entries:
            if e.id == entry_id:
                return e
        raise KeyError(entry_id)


def _check_range(d_min, d_max):
    if not 0 < d_min < d_max:
        raise ValueError(f"need 0 < d_min < d_max, got [{d_min}, {d_max}]")


def _code_of_bits(bits, d_min, d_max, levels):
    """The reference's code of the f32 values with these bit patterns (mapstore.py:112-117)."""
    vals = np.asarray(bits, dtype=np.uint32).view(np.float32).astype(np.float64)
    span = math.log(d_max) - math.log(d_min)
    u = (np.log(np.clip(vals, d_min, d_max)) - math.log(d_min)) / span
    return 1 + np.floor(u * (levels - 1) + 0.5)


@functools.lru_cache(maxsize=32)
def quantize_thresholds(d_min: float, d_max: float, levels: int) -> np.ndarray:
    """f32 [levels-1]: entry k is the smallest f32 depth the reference maps to code k+2.

    Vectorised bisection over positive-f32 bit patterns of the reference's
    formula; a valid depth v then has code 1 + #{thresholds <= v}."""
    _check_range(d_min, d_max)
    n = levels - 1
    if n <= 0:
        return np.zeros(0, dtype=np.float32)
    target = np.arange(2, levels + 1, dtype=np.float64)
    lo = np.ones(n, dtype=np.int64)                      # code(lo) < target (clips to d_min: code 1)
    hi = np.full(n, _F32_MAX_BITS, dtype=np.int64)       # code(hi) == levels >= target
    while True:
        open_ = hi - lo > 1
        if not open_.any():
            break
        mid = (lo + hi) // 2
        ge = _code_of_bits(mid, d_min, d_max, levels) >= target
        hi = np.where(open_ & ge, mid, hi)
        lo = np.where(open_ & ~ge, mid, lo)
    return hi.astype(np.uint32).view(np.float32)


_thr_dev: dict = {}


def _device_thresholds(d_min, d_max, levels):
    import torch
    key = (float(d_min), float(d_max), int(levels), torch.cuda.current_device())
    t = _thr_dev.get(key)
    if t is None:
        thr = quantize_thresholds(float(d_min), float(d_max), int(levels))
        t = torch.from_numpy(np.ascontiguousarray(thr) if thr.size else np.zeros(1, np.float32)).cuda()
        _thr_dev[key] = t
    return t


def _levels_ok(levels):
    if not 1 <= levels <= 65535:
        raise ValueError(f"levels out of range: {levels}")


def quantize_depth_batch(depths, d_min: float = DEFAULT_D_MIN, d_max: float = DEFAULT_D_MAX,
                         levels: int = 255) -> list:
    """``quantize_depth`` of many maps: one H2D, one launch, one D2H."""
    import torch
    _check_range(d_min, d_max)
    levels = int(levels)
    _levels_ok(levels)
    depths = list(depths)
    if not depths:
        return []
    ctx = _lib.context()
    half = [np.asarray(d.values).dtype == np.float16 for d in depths]
    vals = [np.ascontiguousarray(d.values, dtype=np.float16 if h else np.float32) for d, h in zip(depths, half)]
    valid = [np.ascontiguousarray(d.valid, dtype=np.uint8) for d in depths]
    for v, m in zip(vals, valid):
        if v.ndim != 2 or v.shape != m.shape:
            raise ValueError("values and valid must be equal 2-D shapes")
    sizes = [v.size for v in vals]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    tot = int(off[-1])
    # one byte buffer: values (4 B or 2 B per pixel, 16-B aligned per map) then valid masks
    vbytes = [(v.nbytes + 15) & ~15 for v in vals]
    voff = np.concatenate([[0], np.cumsum(vbytes)]).astype(np.int64)
    host = np.zeros(int(voff[-1]) + tot, dtype=np.uint8)
    for k, v in enumerate(vals):
        host[voff[k]:voff[k] + v.nbytes] = v.reshape(-1).view(np.uint8)
    mbase = int(voff[-1])
    for k, m in enumerate(valid):
        host[mbase + off[k]:mbase + off[k + 1]] = m.reshape(-1)
    dev = torch.from_numpy(host).pin_memory().cuda(non_blocking=True)
    out16 = levels > 255
    out = torch.empty(max(tot, 1), dtype=torch.int16 if out16 else torch.uint8, device="cuda")
    esz = 2 if out16 else 1
    jobs = (_lib.DepthCodecJob * len(depths))()
    base = dev.data_ptr()
    for k, v in enumerate(vals):
        j = jobs[k]
        j.height, j.width = v.shape
        j.kind = 1 if half[k] else 0
        j.levels = levels
        j.values = base + int(voff[k])
        j.valid = base + mbase + int(off[k])
        j.out = out.data_ptr() + int(off[k]) * esz
    thr = _device_thresholds(d_min, d_max, levels)
    rc = _lib.lib().vl_quantize_depth(ctx.handle, jobs, len(depths), thr.data_ptr(), levels, _lib.stream_ptr())
    ctx.check(rc, "vl_quantize_depth")
    codes = out.cpu().numpy()
    if out16:
        codes = codes.view(np.uint16)
    res = []
    for k, d in enumerate(depths):
        c = codes[off[k]:off[k + 1]].reshape(vals[k].shape).copy()
        cls = _qclass(d)
        res.append(cls(codes=c, d_min=d_min, d_max=d_max, levels=levels, intrinsics=d.intrinsics))
    return res


def quantize_depth_device(maps, d_min: float = DEFAULT_D_MIN, d_max: float = DEFAULT_D_MAX, levels: int = 255):
    """Device-resident ``quantize_depth`` of many maps in one launch.

    ``maps``: [(depth (h,w) f32 or f16 CUDA tensor, valid (h,w) u8/bool CUDA
    tensor)], e.g. ``DepthBuildPlan.device_maps()``.  Returns code tensors
    ((h,w) uint8, or int16 holding the u16 codes when levels > 255)."""
    import torch
    _check_range(d_min, d_max)
    levels = int(levels)
    _levels_ok(levels)
    maps = list(maps)
    if not maps:
        return []
    ctx = _lib.context()
    sizes = [int(d.numel()) for d, _ in maps]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    out16 = levels > 255
    out = torch.empty(max(int(off[-1]), 1), dtype=torch.int16 if out16 else torch.uint8, device="cuda")
    esz = 2 if out16 else 1
    jobs = (_lib.DepthCodecJob * len(maps))()
    for k, (d, v) in enumerate(maps):
        if d.dim() != 2 or tuple(v.shape) != tuple(d.shape) or not d.is_contiguous() or not v.is_contiguous():
            raise ValueError("values and valid must be equal 2-D contiguous shapes")
        if d.dtype not in (torch.float32, torch.float16) or v.element_size() != 1:
            raise ValueError("depth must be float32/float16 and valid 1 byte per pixel")
        j = jobs[k]
        j.height, j.width = d.shape
        j.kind = 1 if d.dtype == torch.float16 else 0
        j.levels = levels
        j.values = d.data_ptr()
        j.valid = v.data_ptr()
        j.out = out.data_ptr() + int(off[k]) * esz
    thr = _device_thresholds(d_min, d_max, levels)
    rc = _lib.lib().vl_quantize_depth(ctx.handle, jobs, len(maps), thr.data_ptr(), levels, _lib.stream_ptr())
    ctx.check(rc, "vl_quantize_depth")
    return [out[int(off[k]):int(off[k + 1])].view(tuple(maps[k][0].shape)) for k in range(len(maps))]


def _qclass(depth):
    """The QuantizedDepthMap class matching the input's package (reference objects stay reference objects)."""
    mod = type(depth).__module__
    if mod.startswith("visloc."):
        import importlib
        return importlib.import_module("visloc.mapstore").QuantizedDepthMap
    return QuantizedDepthMap


def quantize_depth(depth, d_min: float = DEFAULT_D_MIN, d_max: float = DEFAULT_D_MAX,
                   levels: int = 255) -> QuantizedDepthMap:
    """Drop-in ``mapstore.quantize_depth`` (mapstore.py:96-119), bit-exact codes."""
    return quantize_depth_batch([depth], d_min, d_max, levels)[0]


def _reduce_codes_batch(qs, factor: int, new_levels: int) -> list:
    """Nearest-valid downsample + requantise of many code maps (mapstore.py:390-425)."""
    import torch
    if factor < 1:
        raise ValueError("resolution factors must be >= 1")
    _levels_ok(new_levels)
    if not qs:
        return []
    ctx = _lib.context()
    codes = [np.ascontiguousarray(q.codes) for q in qs]
    nbytes = [(c.nbytes + 15) & ~15 for c in codes]
    ioff = np.concatenate([[0], np.cumsum(nbytes)]).astype(np.int64)
    host = np.zeros(max(int(ioff[-1]), 16), dtype=np.uint8)
    for k, c in enumerate(codes):
        host[ioff[k]:ioff[k] + c.nbytes] = c.reshape(-1).view(np.uint8)
    dev = torch.from_numpy(host).pin_memory().cuda(non_blocking=True)
    shapes = [((c.shape[0] + factor - 1) // factor, (c.shape[1] + factor - 1) // factor) for c in codes]
    out16 = new_levels > 255
    esz = 2 if out16 else 1
    osz = [h * w for h, w in shapes]
    ooff = np.concatenate([[0], np.cumsum(osz)]).astype(np.int64)
    out = torch.empty(max(int(ooff[-1]), 1), dtype=torch.int16 if out16 else torch.uint8, device="cuda")
    jobs = (_lib.DepthCodecJob * len(qs))()
    for k, (q, c) in enumerate(zip(qs, codes)):
        j = jobs[k]
        j.height, j.width = c.shape
        j.kind = 3 if c.dtype == np.uint16 else 2
        j.levels = int(q.levels)
        j.values = dev.data_ptr() + int(ioff[k])
        j.valid = None
        j.out = out.data_ptr() + int(ooff[k]) * esz
    rc = _lib.lib().vl_reduce_depth_codes(ctx.handle, jobs, len(qs), int(factor), int(new_levels),
                                          _lib.stream_ptr())
    ctx.check(rc, "vl_reduce_depth_codes")
    res = out.cpu().numpy()
    if out16:
        res = res.view(np.uint16)
    return [res[ooff[k]:ooff[k + 1]].reshape(shapes[k]).copy() for k in range(len(qs))]


def reduce_depth_codes(q, depth_resolution_factor: int = 1, depth_bits: int = 8):
    """The depth step of ``reduce_map`` for one map: downsample then requantise to
    ``2**depth_bits - 1`` levels (mapstore.py:470-477)."""
    if not 5 <= depth_bits <= 9:
        raise ValueError(f"depth_bits must be within 5..9, got {depth_bits}")
    new_levels = 2 ** depth_bits - 1
    c = _reduce_codes_batch([q], int(depth_resolution_factor), new_levels)[0]
    return type(q)(c, q.d_min, q.d_max, new_levels, q.intrinsics)


def reduce_map(vmap, keyframe_stride: int = 1, rgb_resolution_factor: float = 1.0, rgb_quality: int = 90,
               depth_resolution_factor: int = 1, depth_bits: int = 8):
    """Drop-in ``mapstore.reduce_map`` (mapstore.py:428-497): every kept entry's depth is
    reduced in one GPU launch (per distinct input level count)."""
    if keyframe_stride < 1:
        raise ValueError("keyframe_stride must be >= 1")
    if rgb_resolution_factor < 1 or depth_resolution_factor < 1:
        raise ValueError("resolution factors must be >= 1")
    if not 5 <= depth_bits <= 9:
        raise ValueError(f"depth_bits must be within 5..9, got {depth_bits}")
    if rgb_resolution_factor != 1 or (vmap.rgb_codec != "png" and rgb_quality != 90):
        # RGB re-encoding (mapstore.py:479-490, Pillow) is map storage, outside the
        # hot path: this drop-in reduces depth and keeps RGB payloads
        raise ValueError("RGB resampling / re-encoding is not part of this package (map storage, SURVEY §2); "
                         "use rgb_resolution_factor=1 and the stored codec's quality")
    kept = set(sorted(e.id for e in vmap.entries)[::keyframe_stride])
    entries = [e for e in vmap.entries if e.id in kept]
    new_levels = 2 ** depth_bits - 1
    with_depth = [e for e in entries if e.qdepth is not None]
    reduced = dict(zip((e.id for e in with_depth),
                       _reduce_codes_batch([e.qdepth for e in with_depth], int(depth_resolution_factor),
                                           new_levels)))
    out_entries = []
    for e in entries:
        qd = e.qdepth
        if qd is not None:
            qd = type(qd)(reduced[e.id], qd.d_min, qd.d_max, new_levels, qd.intrinsics)
        out_entries.append(type(e)(id=e.id, pose=e.pose, intrinsics=e.intrinsics, rgb_payload=e.rgb_payload,
                                   rgb_codec=e.rgb_codec, qdepth=qd, descriptor=np.array(e.descriptor, copy=True)))
    return type(vmap)(entries=out_entries, rgb_codec=vmap.rgb_codec, depth_codec=vmap.depth_codec)
