"""ctypes binding of the sm_100a C ABI (include/visloc_b200.h).

The shared library is built in-tree by ``_build.py`` (``__graft_entry__.build``)
and is the only compute path of this package: there is no CPU fallback.  If
the library or a CUDA device is missing every hot-path call raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

import os

# VISLOC_B200_LIB: alternative in-tree build of the same library (A/B kernel experiments)
_LIB_PATH = Path(os.environ.get("VISLOC_B200_LIB") or Path(__file__).resolve().parent / "_lib" / "libvisloc_b200.so")

VL_OK = 0
VL_ERR_INVALID = 1
VL_ERR_CUDA = 2
VL_ERR_OOM = 3
VL_ERR_UNDERCONSTRAINED = 4
VL_ERR_SINGULAR = 5


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double)]


class PCG64State(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64), ("inc_hi", C.c_uint64),
                ("inc_lo", C.c_uint64), ("has_uint32", C.c_uint32), ("uinteger", C.c_uint32)]


class RansacConfigC(C.Structure):
    _fields_ = [("max_iterations", C.c_int64), ("batch_size", C.c_int32), ("max_scoring", C.c_int32),
                ("miss_probability", C.c_double), ("reproj_threshold", C.c_double),
                ("cauchy_scale", C.c_double), ("lm_max_iters", C.c_int32), ("_pad", C.c_int32)]


class RansacArgs(C.Structure):
    _fields_ = [("num_queries", C.c_int32), ("_pad", C.c_int32),
                ("offsets", C.POINTER(C.c_int64)), ("intr", C.POINTER(Intrinsics)),
                ("rng", C.POINTER(PCG64State)), ("px", C.c_void_p), ("X", C.c_void_p),
                ("w", C.c_void_p), ("cfg", RansacConfigC)]


class RansacOut(C.Structure):
    _fields_ = [("q", C.c_void_p), ("t", C.c_void_p), ("inlier_flags", C.c_void_p),
                ("inlier_count", C.c_void_p), ("score", C.c_void_p), ("iterations", C.c_void_p),
                ("converged", C.c_void_p), ("stats", C.c_void_p)]


class DepthCodecJob(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("kind", C.c_int32), ("levels", C.c_int32),
                ("values", C.c_void_p), ("valid", C.c_void_p), ("out", C.c_void_p)]


class TriView(C.Structure):
    _fields_ = [("targets", C.c_void_p), ("confidence", C.c_void_p), ("rt", C.c_double * 9),
                ("center", C.c_double * 3), ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double),
                ("cy", C.c_double)]


class TriMap(C.Structure):
    _fields_ = [("grid_w", C.c_int32), ("grid_h", C.c_int32), ("view0", C.c_int32), ("nview", C.c_int32),
                ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("sx", C.c_double), ("sy", C.c_double), ("R", C.c_double * 9), ("center", C.c_double * 3),
                ("depth", C.c_void_p), ("valid", C.c_void_p)]


class TriConfig(C.Structure):
    _fields_ = [("angular_threshold_rad", C.c_double), ("confidence_threshold", C.c_double),
                ("refine_tol", C.c_double), ("min_inliers", C.c_int32), ("max_refine_iters", C.c_int32)]


class TriProblem(C.Structure):
    _fields_ = [("ray", C.c_double * 3), ("center", C.c_double * 3), ("obs0", C.c_int32), ("nobs", C.c_int32)]


class TriObs(C.Structure):
    _fields_ = [("rt", C.c_double * 9), ("center", C.c_double * 3), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("target", C.c_double * 2), ("confidence", C.c_double)]


ctypes_ref = C.byref

LIFT_PLANAR, LIFT_IMLC = 0, 1
FIELD_BAD_CONF, FIELD_BAD_TARGET = 1, 2


class LiftSegment(C.Structure):
    _fields_ = [("query", C.c_int32), ("entry", C.c_int32), ("direction", C.c_int32), ("depth", C.c_int32),
                ("grid_w", C.c_int32), ("grid_h", C.c_int32), ("layout", C.c_int32), ("_pad", C.c_int32),
                ("scale_x", C.c_double), ("scale_y", C.c_double),
                ("targets", C.c_void_p), ("confidence", C.c_void_p)]


# numpy view of an array of vl_lift_segment (vectorised segment tables)
LIFT_SEGMENT_DTYPE = np.dtype([("query", "<i4"), ("entry", "<i4"), ("direction", "<i4"), ("depth", "<i4"),
                               ("grid_w", "<i4"), ("grid_h", "<i4"), ("layout", "<i4"), ("_pad", "<i4"),
                               ("scale_x", "<f8"), ("scale_y", "<f8"), ("targets", "<u8"),
                               ("confidence", "<u8")])
assert LIFT_SEGMENT_DTYPE.itemsize == C.sizeof(LiftSegment)

IMLC_OK, IMLC_MAGIC, IMLC_VERSION, IMLC_TRUNCATED, IMLC_TRAILING = 0, 1, 2, 3, 4


class ImlcHeader(C.Structure):
    _fields_ = [("status", C.c_int32), ("version", C.c_uint32), ("error_offset", C.c_int64),
                ("need", C.c_int64), ("have", C.c_int64), ("what", C.c_char_p), ("magic", C.c_uint8 * 4),
                ("grid_w", C.c_uint32), ("grid_h", C.c_uint32), ("scale_x", C.c_double), ("scale_y", C.c_double),
                ("source_off", C.c_int64), ("source_len", C.c_int64), ("target_off", C.c_int64),
                ("target_len", C.c_int64), ("records_off", C.c_int64)]


class LiftDepth(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("kind", C.c_int32), ("_pad", C.c_int32),
                ("values", C.c_void_p), ("valid", C.c_void_p), ("lut", C.c_void_p),
                ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("sx_depth", C.c_double), ("sy_depth", C.c_double),
                ("R", C.c_double * 9), ("t", C.c_double * 3)]


class VislocError(RuntimeError):
    pass


_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load the shared library (once); raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not _LIB_PATH.exists():
            raise VislocError(
                f"{_LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                "There is no CPU fallback.")
        L = C.CDLL(str(_LIB_PATH))
        vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int32)
        L.vl_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.vl_destroy.argtypes = [vp]
        L.vl_last_error.argtypes = [vp]
        L.vl_last_error.restype = C.c_char_p
        L.vl_launch_count.argtypes = [vp]
        L.vl_launch_count.restype = i64
        L.vl_reserve.argtypes = [vp, i32, i64, i32]
        L.vl_pcg64_seed.argtypes = [C.c_uint64, C.POINTER(PCG64State)]
        L.vl_profile.argtypes = [vp, C.c_int]
        L.vl_profile_read.argtypes = [vp, dp, C.POINTER(C.c_int64), i32]
        L.vl_ransac_pnp.argtypes = [vp, C.POINTER(RansacArgs), C.POINTER(RansacOut), vp]
        L.vl_msac_score.argtypes = [vp, dp, dp, vp, vp, vp, i64, Intrinsics, dbl, dp, vp, vp]
        L.vl_score_hypotheses.argtypes = [vp, vp, vp, i32, vp, vp, vp, i64, Intrinsics, dbl, i32, vp, vp]
        L.vl_score_hypotheses.restype = C.c_int
        L.vl_set_scoring_pruning.argtypes = [vp, i32]
        L.vl_set_scoring_pruning.restype = C.c_int
        L.vl_scoring_counters.argtypes = [vp, C.POINTER(C.c_int64), i32]
        L.vl_scoring_counters.restype = C.c_int
        L.vl_refine_pose.argtypes = [vp, dp, dp, vp, vp, vp, i64, Intrinsics, i32, dbl, i32, dbl, dbl,
                                     ip, ip, dp, ip, vp]
        L.vl_p3p_solve_batch.argtypes = [vp, vp, vp, i32, vp, vp, vp, ip, vp]
        L.vl_sample_minimal_sets.argtypes = [vp, C.POINTER(PCG64State), i64, i32, vp, vp]
        L.vl_lift.argtypes = [vp, vp, i32, C.POINTER(LiftDepth), i32, i32, dbl, i32,
                              vp, vp, vp, vp, i64, C.POINTER(C.c_int64), C.POINTER(C.c_int32), vp]
        L.vl_imlc_parse.argtypes = [vp, i64, C.POINTER(ImlcHeader)]
        L.vl_retrieval_topk.argtypes = [vp, vp, vp, i32, i32, vp, i32, i32, vp, vp, vp]
        L.vl_ransac_pnp_staged.argtypes = [vp, C.POINTER(RansacArgs), C.POINTER(RansacOut), i32,
                                           C.POINTER(C.c_int32), C.POINTER(vp), vp]
        L.vl_ransac_pnp_staged.restype = C.c_int
        L.vl_retrieval_topk.restype = C.c_int
        L.vl_imlc_parse.restype = C.c_int
        L.vl_interp_depth.argtypes = [vp, C.POINTER(LiftDepth), vp, i64, vp, vp, vp]
        L.vl_decode_depth.argtypes = [vp, C.POINTER(LiftDepth), vp, vp, vp]
        L.vl_robust_cost.argtypes = [vp, dp, dp, vp, vp, vp, i64, Intrinsics, i32, dbl, dp, vp]
        L.vl_pose_residuals.argtypes = [vp, dp, dp, vp, vp, i64, Intrinsics, vp, vp, vp, vp]
        L.vl_ransac_begin.argtypes = [vp, C.POINTER(RansacArgs), i32, i32, vp]
        L.vl_ransac_partial_bytes.argtypes = [vp, C.POINTER(C.c_int64)]
        L.vl_ransac_step_score.argtypes = [vp, vp, vp]
        L.vl_ransac_step_finish.argtypes = [vp, vp, C.POINTER(C.c_int32), vp]
        L.vl_ransac_end.argtypes = [vp, C.POINTER(RansacOut), vp]
        L.vl_ransac_step_argmin.argtypes = [vp, vp, vp]
        L.vl_ransac_step_finish_argmin.argtypes = [vp, vp, C.POINTER(C.c_int32), vp]
        for name in ("vl_ransac_begin", "vl_ransac_partial_bytes", "vl_ransac_step_score",
                     "vl_ransac_step_finish", "vl_ransac_end", "vl_ransac_step_argmin",
                     "vl_ransac_step_finish_argmin"):
            getattr(L, name).restype = C.c_int
        L.vl_quantize_depth.argtypes = [vp, C.POINTER(DepthCodecJob), i32, vp, i32, vp]
        L.vl_reduce_depth_codes.argtypes = [vp, C.POINTER(DepthCodecJob), i32, i32, i32, vp]
        L.vl_quantize_depth.restype = C.c_int
        L.vl_reduce_depth_codes.restype = C.c_int
        L.vl_build_depth_maps.argtypes = [vp, C.POINTER(TriMap), i32, C.POINTER(TriView), i32, i32,
                                          C.POINTER(TriConfig), vp]
        L.vl_triangulate_rays.argtypes = [vp, vp, i32, vp, i32, C.POINTER(TriConfig), vp, vp, vp, vp]
        L.vl_build_depth_maps.restype = C.c_int
        L.vl_triangulate_rays.restype = C.c_int
        L.vl_robust_cost.restype = C.c_int
        L.vl_pose_residuals.restype = C.c_int
        for name in ("vl_create", "vl_destroy", "vl_reserve", "vl_pcg64_seed", "vl_ransac_pnp", "vl_profile",
                     "vl_profile_read", "vl_lift", "vl_interp_depth", "vl_decode_depth",
                     "vl_msac_score", "vl_refine_pose", "vl_p3p_solve_batch", "vl_sample_minimal_sets"):
            getattr(L, name).restype = C.c_int
        _lib = L
        return L


EXPORTED_SYMBOLS = (
    "vl_create", "vl_destroy", "vl_last_error", "vl_reserve", "vl_launch_count", "vl_pcg64_seed",
    "vl_ransac_pnp", "vl_msac_score", "vl_refine_pose", "vl_p3p_solve_batch",
    "vl_sample_minimal_sets", "vl_profile", "vl_profile_read", "vl_lift", "vl_interp_depth",
    "vl_decode_depth", "vl_robust_cost", "vl_pose_residuals", "vl_ransac_begin", "vl_ransac_partial_bytes",
    "vl_ransac_step_score", "vl_ransac_step_finish", "vl_ransac_end", "vl_imlc_parse",
    "vl_retrieval_topk", "vl_ransac_pnp_staged", "vl_quantize_depth", "vl_reduce_depth_codes",
    "vl_build_depth_maps", "vl_triangulate_rays", "vl_ransac_step_argmin", "vl_ransac_step_finish_argmin",
    "vl_score_hypotheses", "vl_set_scoring_pruning", "vl_scoring_counters",
)

STAGES = ("prep", "sample", "p3p", "compact", "score", "scan", "active", "final", "lift")


class Context:
    """One C-ABI context per CUDA device (workspace lives here)."""

    def __init__(self, device: int):
        self.device = device
        self.handle = C.c_void_p()
        rc = lib().vl_create(device, C.byref(self.handle))
        if rc != VL_OK:
            raise VislocError(f"vl_create(device={device}) failed with status {rc} "
                              "(a B200 / sm_100 GPU is required)")

    def check(self, rc: int, what: str):
        if rc == VL_OK:
            return
        msg = lib().vl_last_error(self.handle).decode(errors="replace")
        if rc == VL_ERR_INVALID:
            raise ValueError(f"{what}: {msg}")
        if rc == VL_ERR_UNDERCONSTRAINED:
            from .posest import UnderConstrainedError
            raise UnderConstrainedError(msg)
        if rc == VL_ERR_SINGULAR:
            raise ValueError(msg)
        raise VislocError(f"{what} failed ({rc}): {msg}")

    def launches(self) -> int:
        return int(lib().vl_launch_count(self.handle))

    def set_pruning(self, enable: bool):
        """Exact scoring pruning on / off (vl_set_scoring_pruning; outputs identical either way)."""
        self.check(lib().vl_set_scoring_pruning(self.handle, 1 if enable else 0), "vl_set_scoring_pruning")

    def scoring_counters(self, reset: bool = False) -> tuple[int, int]:
        """(evaluations skipped by pruning, evaluations done by the tail pass) since the last reset."""
        out = (C.c_int64 * 2)()
        self.check(lib().vl_scoring_counters(self.handle, out, 1 if reset else 0), "vl_scoring_counters")
        return int(out[0]), int(out[1])

    def profile(self, enable: bool):
        lib().vl_profile(self.handle, 1 if enable else 0)

    def profile_read(self) -> dict:
        ms = (C.c_double * len(STAGES))()
        cnt = (C.c_int64 * len(STAGES))()
        lib().vl_profile_read(self.handle, ms, cnt, len(STAGES))
        return {s: (float(ms[i]), int(cnt[i])) for i, s in enumerate(STAGES)}

    def __del__(self):
        try:
            if self.handle:
                lib().vl_destroy(self.handle)
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    import torch
    if not torch.cuda.is_available():
        raise VislocError("CUDA device not available: the visloc_b200 hot path runs only on the GPU")
    if device is None:
        device = torch.cuda.current_device()
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        _contexts[device] = ctx
    return ctx


def pcg64_state(seed: int) -> PCG64State:
    """numpy ``default_rng(seed)`` generator state (C implementation for 0 <= seed < 2^64)."""
    st = PCG64State()
    if 0 <= int(seed) < 2 ** 64:
        rc = lib().vl_pcg64_seed(C.c_uint64(int(seed)), C.byref(st))
        if rc != VL_OK:
            raise ValueError(f"bad seed {seed}")
        return st
    # arbitrary-precision seeds: numpy's own SeedSequence (host-side seeding only)
    s = np.random.PCG64(int(seed)).state
    return state_from_numpy(s)


def state_from_numpy(s: dict) -> PCG64State:
    st = PCG64State()
    v, inc = int(s["state"]["state"]), int(s["state"]["inc"])
    m64 = (1 << 64) - 1
    st.state_hi, st.state_lo = v >> 64, v & m64
    st.inc_hi, st.inc_lo = inc >> 64, inc & m64
    st.has_uint32 = int(s["has_uint32"])
    st.uinteger = int(s["uinteger"])
    return st


def state_to_dict(st: PCG64State) -> dict:
    return {"state": (int(st.state_hi) << 64) | int(st.state_lo),
            "inc": (int(st.inc_hi) << 64) | int(st.inc_lo),
            "has_uint32": int(st.has_uint32), "uinteger": int(st.uinteger)}


def stream_ptr():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def nvtx(name: str):
    """NVTX range around a host API stage (visible in Nsight Systems / ncu
    --nvtx); a no-op context when NVTX is unavailable."""
    import contextlib
    try:
        import torch
        return torch.cuda.nvtx.range(name)
    except Exception:  # pragma: no cover
        return contextlib.nullcontext()
