"""LM pose refinement — drop-in for ``visloc.refine`` (refine.py:1-230).

``refine_pose`` runs the whole Levenberg-Marquardt loop in one CTA on the
GPU (``vl_refine_pose``): fused cost / gradient / J^T W J passes with
deterministic block reductions, the reference's damping schedule
(lambda 1e-6, 25 trials x10, /3 floor 1e-12) and stopping rules.  Losses and
``apply_delta`` are small host-side values mirroring the reference.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .geometry import CameraIntrinsics, Pose, quat_multiply, rotvec_to_quat

__all__ = ["CauchyLoss", "RefineResult", "TruncatedLoss", "apply_delta", "pose_jacobian", "pose_residuals",
           "refine_pose", "robust_cost"]


@dataclass(frozen=True)
class TruncatedLoss:
    tau: float

    def __post_init__(self):
        if self.tau <= 0:
            raise ValueError("tau must be positive")

    def rho(self, e2):
        return np.minimum(e2, self.tau * self.tau)

    def weight(self, e2):
        return (np.asarray(e2) < self.tau * self.tau).astype(np.float64)

    def behind_cost(self) -> float:
        return self.tau * self.tau


@dataclass(frozen=True)
class CauchyLoss:
    scale: float

    def __post_init__(self):
        if self.scale <= 0:
            raise ValueError("scale must be positive")

    def rho(self, e2):
        c2 = self.scale * self.scale
        return 0.5 * c2 * np.log1p(np.asarray(e2) / c2)

    def weight(self, e2):
        return 0.5 / (1.0 + np.asarray(e2) / (self.scale * self.scale))

    def behind_cost(self) -> float:
        return math.inf


def apply_delta(pose: Pose, delta) -> Pose:
    """Left-compose (omega, nu) onto a pose (refine.py:80-87)."""
    omega = np.asarray(delta[:3], dtype=np.float64)
    nu = np.asarray(delta[3:6], dtype=np.float64)
    dq = rotvec_to_quat(omega)
    q = quat_multiply(dq, pose.q)
    return Pose(q, Pose(dq, np.zeros(3)).R @ pose.t + nu)


def _loss_kind(loss):
    if isinstance(loss, TruncatedLoss):
        return 0, float(loss.tau)
    if isinstance(loss, CauchyLoss):
        return 1, float(loss.scale)
    # duck-typed reference losses
    if hasattr(loss, "tau"):
        return 0, float(loss.tau)
    if hasattr(loss, "scale"):
        return 1, float(loss.scale)
    raise TypeError(f"unsupported loss {type(loss).__name__}")


def _pose_ptrs(pose):
    q = np.ascontiguousarray(pose.q, dtype=np.float64)
    t = np.ascontiguousarray(pose.t, dtype=np.float64)
    dp = C.POINTER(C.c_double)
    return q, t, q.ctypes.data_as(dp), t.ctypes.data_as(dp)


def robust_cost(pose: Pose, points, pixels, weights, loss, intr: CameraIntrinsics) -> float:
    """Weighted robust cost (refine.py:135-149), one fused GPU pass."""
    from .posest import _intr_c, _to_device
    X = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    px = np.ascontiguousarray(np.asarray(pixels, dtype=np.float64).reshape(-1, 2))
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).reshape(-1))
    kind, scale = _loss_kind(loss)
    ctx = _lib.context()
    dX, dpx, dw = _to_device(X), _to_device(px), _to_device(w)
    q, t, qp, tp = _pose_ptrs(pose)
    out = C.c_double()
    rc = _lib.lib().vl_robust_cost(ctx.handle, qp, tp, dpx.data_ptr(), dX.data_ptr(), dw.data_ptr(), X.shape[0],
                                   _intr_c(intr), kind, scale, C.byref(out), _lib.stream_ptr())
    ctx.check(rc, "vl_robust_cost")
    return float(out.value)


def _residuals_gpu(pose, points, pixels, intr, want_res, want_J):
    import torch
    from .posest import _intr_c, _to_device
    X = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    n = X.shape[0]
    px = np.ascontiguousarray(np.asarray(pixels, dtype=np.float64).reshape(-1, 2)) if pixels is not None \
        else np.zeros((n, 2))
    ctx = _lib.context()
    dX, dpx = _to_device(X), _to_device(px)
    res = torch.empty((max(n, 1), 2), dtype=torch.float64, device="cuda")
    z = torch.empty((max(n, 1),), dtype=torch.float64, device="cuda")
    J = torch.empty((max(n, 1), 2, 6), dtype=torch.float64, device="cuda") if want_J else None
    q, t, qp, tp = _pose_ptrs(pose)
    rc = _lib.lib().vl_pose_residuals(ctx.handle, qp, tp, dpx.data_ptr(), dX.data_ptr(), n, _intr_c(intr),
                                      res.data_ptr(), z.data_ptr(), J.data_ptr() if J is not None else None,
                                      _lib.stream_ptr())
    ctx.check(rc, "vl_pose_residuals")
    return res[:n].cpu().numpy(), z[:n].cpu().numpy(), (J[:n].cpu().numpy() if J is not None else None)


def pose_residuals(pose: Pose, points, pixels, intr: CameraIntrinsics):
    """Reprojection residuals (N,2) and camera-frame z (N,) (refine.py:90-100)."""
    r, z, _ = _residuals_gpu(pose, points, pixels, intr, True, False)
    return r, z


def pose_jacobian(pose: Pose, points, intr: CameraIntrinsics) -> np.ndarray:
    """Analytic residual Jacobian (N,2,6) at delta = 0, rows zeroed at/behind the camera (refine.py:103-132)."""
    _, _, J = _residuals_gpu(pose, points, None, intr, False, True)
    return J


@dataclass
class RefineResult:
    pose: Pose
    converged: bool
    iterations: int
    cost_trace: list = field(default_factory=list)

    @property
    def final_cost(self) -> float:
        return self.cost_trace[-1] if self.cost_trace else math.nan


def refine_pose(initial: Pose, points, pixels, weights, loss, intr: CameraIntrinsics,
                max_iters: int = 100, gradient_tol: float = 1e-10,
                cost_tol: float = 1e-12) -> RefineResult:
    """LM minimisation of the weighted robust reprojection cost (refine.py:164-230)."""
    from .posest import _to_device
    X = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    px = np.ascontiguousarray(np.asarray(pixels, dtype=np.float64).reshape(-1, 2))
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).reshape(-1))
    if X.shape[0] < 3:
        raise ValueError(f"refinement needs >= 3 matches, got {X.shape[0]}")
    kind, scale = _loss_kind(loss)
    ctx = _lib.context()
    dX, dpx, dw = _to_device(X), _to_device(px), _to_device(w)
    q = np.ascontiguousarray(initial.q, dtype=np.float64).copy()
    t = np.ascontiguousarray(initial.t, dtype=np.float64).copy()
    trace = np.zeros(max(int(max_iters), 0) + 1, dtype=np.float64)
    conv, iters, tlen = C.c_int32(), C.c_int32(), C.c_int32()
    dp = C.POINTER(C.c_double)
    from .posest import _intr_c
    rc = _lib.lib().vl_refine_pose(
        ctx.handle, q.ctypes.data_as(dp), t.ctypes.data_as(dp), dpx.data_ptr(), dX.data_ptr(),
        dw.data_ptr(), X.shape[0], _intr_c(intr), kind, scale, int(max_iters), float(gradient_tol),
        float(cost_tol), C.byref(conv), C.byref(iters), trace.ctypes.data_as(dp), C.byref(tlen),
        _lib.stream_ptr())
    ctx.check(rc, "vl_refine_pose")
    return RefineResult(pose=Pose(q, t), converged=bool(conv.value), iterations=int(iters.value),
                        cost_trace=[float(c) for c in trace[:tlen.value]])
