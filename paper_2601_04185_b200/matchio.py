"""Correspondence fields and the IMLC exchange format — drop-in for ``visloc.matchio``.

Two ways in:

* ``read_field`` / ``write_field`` / ``CorrespondenceField`` /
  ``filter_matches_arrays`` behave like the reference (matchio.py:74-218):
  a parsed field is a host numpy object.
* ``FieldArena`` is the B200 ingestion path: many IMLC
  blobs packed back to back in ONE pinned host buffer (read straight from
  files or sockets), headers parsed in C (``vl_imlc_parse``, the reference's
  validation order and error offsets), one host-to-device copy, and the lift
  kernels read the 12-byte records in place — no per-field numpy objects.
  Record content (confidence finite in [0, 1], finite targets where
  confidence > 0) is validated on the GPU by the same pass that counts the
  gated cells; a violation raises the reference's ``FieldFormatError``
  ("invalid field content: ...") when the field is lifted.

Layout (little-endian, matchio.py:9-20): ``b"IMLC"``, u32 version (1),
u32 + UTF-8 source id, u32 + UTF-8 target id, u32 grid_w, u32 grid_h,
f64 scale_x, f64 scale_y, then grid_h*grid_w records (x f32, y f32, conf f32).
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib

__all__ = [
    "CorrespondenceField", "FieldArena", "FieldBlob", "FieldFormatError", "FieldMagicError",
    "FieldTruncatedError", "FieldVersionError", "FilteredMatch", "MAGIC", "VERSION", "field_bytes", "filter_matches",
    "filter_matches_arrays",
    "parse_header", "read_field", "read_field_blob", "write_field",
]

MAGIC = b"IMLC"
VERSION = 1


class FieldFormatError(ValueError):
    """Malformed field file; ``offset`` is the byte position of the problem."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (at byte offset {offset})")
        self.offset = offset


class FieldMagicError(FieldFormatError):
    pass


class FieldVersionError(FieldFormatError):
    pass


class FieldTruncatedError(FieldFormatError):
    pass


@dataclass
class CorrespondenceField:
    """Per-cell targets (h,w,2) and confidences (h,w) (matchio.py:74-123)."""

    source_id: str
    target_id: str
    targets: np.ndarray
    confidence: np.ndarray
    scale_x: float = 1.0
    scale_y: float = 1.0

    def __post_init__(self):
        t32 = np.asarray(self.targets).dtype == np.float32
        c32 = np.asarray(self.confidence).dtype == np.float32
        self.targets = np.ascontiguousarray(self.targets, dtype=np.float32 if t32 else np.float64)
        self.confidence = np.ascontiguousarray(self.confidence, dtype=np.float32 if c32 else np.float64)
        if self.targets.ndim != 3 or self.targets.shape[2] != 2:
            raise ValueError(f"targets must be (H, W, 2), got {self.targets.shape}")
        if self.confidence.shape != self.targets.shape[:2]:
            raise ValueError(f"confidence shape {self.confidence.shape} does not match "
                             f"targets {self.targets.shape[:2]}")
        h, w = self.confidence.shape
        if h <= 0 or w <= 0:
            raise ValueError(f"grid dimensions must be positive, got {w}x{h}")
        c = self.confidence
        if np.any(~np.isfinite(c)) or c.min() < 0 or c.max() > 1:
            raise ValueError("confidences must be finite and within [0, 1]")
        if np.any(~np.isfinite(self.targets[c > 0])):
            raise ValueError("matched cells (confidence > 0) must have finite targets")

    @property
    def grid_w(self) -> int:
        return self.confidence.shape[1]

    @property
    def grid_h(self) -> int:
        return self.confidence.shape[0]


# ----------------------------------------------------------------------------- writer
def field_bytes(field) -> bytes:
    """IMLC serialization of a field (matchio.write_field, :136-156)."""
    src = field.source_id.encode("utf-8")
    tgt = field.target_id.encode("utf-8")
    records = np.empty((field.grid_h, field.grid_w, 3), dtype="<f4")
    records[..., :2] = field.targets
    records[..., 2] = field.confidence
    return b"".join([MAGIC, struct.pack("<I", VERSION), struct.pack("<I", len(src)), src,
                     struct.pack("<I", len(tgt)), tgt, struct.pack("<II", field.grid_w, field.grid_h),
                     struct.pack("<dd", field.scale_x, field.scale_y), records.tobytes()])


def write_field(field, destination) -> None:
    """Serialize a field; ``read_field`` of the result is bit-exact."""
    Path(destination).write_bytes(field_bytes(field))


# ----------------------------------------------------------------------------- header parse
@dataclass(frozen=True)
class ImlcInfo:
    """Parsed IMLC header; byte offsets are relative to the blob start."""

    source_id: str
    target_id: str
    grid_w: int
    grid_h: int
    scale_x: float
    scale_y: float
    records_off: int
    nbytes: int


def _as_u8(buf) -> np.ndarray:
    if isinstance(buf, np.ndarray):
        return np.ascontiguousarray(buf).view(np.uint8).reshape(-1)
    return np.frombuffer(memoryview(buf).cast("B"), dtype=np.uint8)


def parse_header(buf) -> ImlcInfo:
    """Validate an IMLC blob's framing (vl_imlc_parse) and return its header.

    Raises the reference's errors with its messages and offsets
    (matchio.py:160-190); record content is not checked here."""
    a = _as_u8(buf)
    h = _lib.ImlcHeader()
    rc = _lib.lib().vl_imlc_parse(a.ctypes.data if a.size else None, int(a.size), C.byref(h))
    if rc != _lib.VL_OK:
        raise ValueError("vl_imlc_parse: bad arguments")
    if h.status == _lib.IMLC_TRUNCATED:
        what = h.what.decode()
        need = int(h.need) if h.need >= 0 else 12 * int(h.grid_w) * int(h.grid_h)
        raise FieldTruncatedError(f"truncated file: need {need} bytes for {what}, have {int(h.have)}",
                                  int(h.error_offset))
    if h.status == _lib.IMLC_MAGIC:
        raise FieldMagicError(f"bad magic {bytes(h.magic)!r}, expected {MAGIC!r}", 0)
    if h.status == _lib.IMLC_VERSION:
        raise FieldVersionError(f"unsupported version {int(h.version)}, expected {VERSION}", 4)
    if h.status == _lib.IMLC_TRAILING:
        raise FieldFormatError(f"{int(h.have)} trailing bytes after records", int(h.error_offset))
    raw = a.data.cast("B") if a.size else memoryview(b"")
    src = bytes(raw[h.source_off:h.source_off + h.source_len]).decode("utf-8")
    tgt = bytes(raw[h.target_off:h.target_off + h.target_len]).decode("utf-8")
    info = ImlcInfo(src, tgt, int(h.grid_w), int(h.grid_h), float(h.scale_x), float(h.scale_y),
                    int(h.records_off), int(a.size))
    if info.grid_w <= 0 or info.grid_h <= 0:  # CorrespondenceField.__post_init__ (:97-99)
        raise FieldFormatError(f"invalid field content: grid dimensions must be positive, got "
                               f"{info.grid_w}x{info.grid_h}", info.records_off)
    return info


def read_field(source) -> CorrespondenceField:
    """Parse an IMLC file into a host ``CorrespondenceField`` (matchio.read_field)."""
    data = Path(source).read_bytes()
    info = parse_header(data)
    n = info.grid_w * info.grid_h
    records = np.frombuffer(data, dtype="<f4", count=3 * n, offset=info.records_off).reshape(
        info.grid_h, info.grid_w, 3).copy()
    try:
        return CorrespondenceField(source_id=info.source_id, target_id=info.target_id,
                                   targets=records[..., :2], confidence=records[..., 2],
                                   scale_x=info.scale_x, scale_y=info.scale_y)
    except ValueError as exc:
        raise FieldFormatError(f"invalid field content: {exc}", len(data) - 12 * n) from exc


# ----------------------------------------------------------------------------- arena
class FieldBlob:
    """One IMLC field inside a ``FieldArena`` (duck-types CorrespondenceField).

    ``targets`` / ``confidence`` are zero-copy numpy views of the pinned
    records (for host-side consumers); the GPU lift reads the records in
    place (``vl_lift`` layout ``VL_LIFT_IMLC``)."""

    __slots__ = ("arena", "index", "info", "start")

    def __init__(self, arena, index: int, info: ImlcInfo, start: int):
        self.arena, self.index, self.info, self.start = arena, index, info, start

    source_id = property(lambda self: self.info.source_id)
    target_id = property(lambda self: self.info.target_id)
    grid_w = property(lambda self: self.info.grid_w)
    grid_h = property(lambda self: self.info.grid_h)
    scale_x = property(lambda self: self.info.scale_x)
    scale_y = property(lambda self: self.info.scale_y)

    @property
    def records_offset(self) -> int:
        """Byte offset of the first record inside the arena (4-byte aligned)."""
        return self.start + self.info.records_off

    def records(self) -> np.ndarray:
        n = self.grid_w * self.grid_h
        return self.arena.host_u8[self.records_offset:self.records_offset + 12 * n].view("<f4").reshape(
            self.grid_h, self.grid_w, 3)

    @property
    def targets(self) -> np.ndarray:
        return self.records()[..., :2]

    @property
    def confidence(self) -> np.ndarray:
        return self.records()[..., 2]

    def to_field(self) -> CorrespondenceField:
        """Host ``CorrespondenceField`` copy (reference object path, validated)."""
        r = self.records().copy()
        try:
            return CorrespondenceField(self.source_id, self.target_id, r[..., :2], r[..., 2],
                                       self.scale_x, self.scale_y)
        except ValueError as exc:
            raise FieldFormatError(f"invalid field content: {exc}", self.info.records_off) from exc

    def content_error(self, flags: int) -> FieldFormatError:
        msg = ("confidences must be finite and within [0, 1]" if flags & _lib.FIELD_BAD_CONF
               else "matched cells (confidence > 0) must have finite targets")
        return FieldFormatError(f"invalid field content: {msg}", self.info.records_off)


class FieldArena:
    """Many IMLC blobs in one pinned host buffer, mirrored to HBM with one copy.

    Each blob is placed so its records start 16-byte aligned.  ``blobs`` are
    bytes-like objects or file paths (read straight into the pinned buffer).
    Framing errors raise like ``read_field`` at construction."""

    def __init__(self, blobs):
        import torch
        items = list(blobs)
        sizes, paths = [], []
        for b in items:
            if isinstance(b, (str, Path)):
                p = Path(b)
                paths.append(p)
                sizes.append(p.stat().st_size)
            else:
                paths.append(None)
                sizes.append(memoryview(b).nbytes)
        # first pass over the headers to place every records region on a 16-B boundary
        heads = []
        for b, p in zip(items, paths):
            if p is not None:
                with open(p, "rb") as fh:
                    head = fh.read(4096)
            else:
                head = bytes(memoryview(b).cast("B")[:4096])
            heads.append(head)
        pre = [self._records_off_hint(h) for h in heads]
        starts, pos = [], 0
        for s, r in zip(sizes, pre):
            pos += (-(pos + r)) % 16
            starts.append(pos)
            pos += s
        self.nbytes = pos
        self.host = torch.empty(max(pos, 16), dtype=torch.uint8, pin_memory=True)
        self.host_u8 = self.host.numpy()
        for b, p, st, s in zip(items, paths, starts, sizes):
            dst = self.host_u8[st:st + s]
            if p is not None:
                with open(p, "rb") as fh:
                    fh.readinto(memoryview(dst))
            else:
                dst[:] = _as_u8(b)
        self.fields = []
        for i, (st, s) in enumerate(zip(starts, sizes)):
            info = parse_header(self.host_u8[st:st + s])
            self.fields.append(FieldBlob(self, i, info, st))
        # per-field geometry as arrays (vectorised segment tables)
        self.gw = np.array([f.info.grid_w for f in self.fields], dtype=np.int64)
        self.gh = np.array([f.info.grid_h for f in self.fields], dtype=np.int64)
        self.sx = np.array([f.info.scale_x for f in self.fields], dtype=np.float64)
        self.sy = np.array([f.info.scale_y for f in self.fields], dtype=np.float64)
        self.roff = np.array([f.start + f.info.records_off for f in self.fields], dtype=np.uint64)
        self._dev = None
        self.ready = None

    @staticmethod
    def _records_off_hint(head: bytes) -> int:
        try:
            ls = struct.unpack_from("<I", head, 8)[0]
            lt = struct.unpack_from("<I", head, 12 + ls)[0]
            return 12 + ls + 4 + lt + 24
        except struct.error:
            return 0

    def __len__(self):
        return len(self.fields)

    def __getitem__(self, i) -> FieldBlob:
        return self.fields[i]

    def device(self, stream=None):
        """HBM mirror of the arena (one host-to-device copy, issued once)."""
        import torch
        if self._dev is None:
            dev = torch.empty_like(self.host, device="cuda")
            with torch.cuda.stream(stream) if stream is not None else _nullctx():
                dev.copy_(self.host, non_blocking=True)
            self._dev = dev
        return self._dev

    def upload(self, out, stream=None):
        """Copy the arena into a caller-owned uint8 CUDA tensor (>= nbytes) and use it.

        With a side ``stream`` the copy overlaps whatever the caller does next
        (retrieval, planning); consumers (the lift) wait on ``ready``."""
        import torch
        self.ready = None
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            out[: self.host.numel()].copy_(self.host, non_blocking=True)
            if stream is not None:
                self.ready = torch.cuda.Event()
                self.ready.record(stream)
        self._dev = out
        return out

    def wait(self, stream=None):
        """Make `stream` (default: current) wait for the arena's device copy."""
        import torch
        if getattr(self, "ready", None) is not None:
            (stream or torch.cuda.current_stream()).wait_event(self.ready)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def read_field_blob(source) -> FieldBlob:
    """One IMLC blob (bytes or path) as a single-field arena."""
    return FieldArena([source])[0]


def filter_matches_arrays(fld, threshold: float):
    """(source_px (M,2), target_px (M,2), confidence (M,), flat cell index (M,)) on the GPU
    (matchio.py:203-218)."""
    from .localizer import _run_lift
    px, X, w, _, _, _ = _run_lift([(0, 0, 0, 0, fld)], [], threshold, mode=1)
    Xh = X.cpu().numpy()
    return px.cpu().numpy(), Xh[:, :2].copy(), w.cpu().numpy(), Xh[:, 2].astype(np.int64)


@dataclass
class FilteredMatch:
    """A confidence-gated match in source/target pixel coordinates (matchio.py:127-132)."""

    source_px: np.ndarray
    target_px: np.ndarray
    confidence: float


def filter_matches(fld, threshold: float) -> list[FilteredMatch]:
    """Per-match view of ``filter_matches_arrays`` (matchio.py:221-228): cells with
    confidence >= threshold and > 0, row-major, gated on the GPU."""
    src, tgt, conf, _ = filter_matches_arrays(fld, threshold)
    return [FilteredMatch(src[i], tgt[i], float(conf[i])) for i in range(len(conf))]
