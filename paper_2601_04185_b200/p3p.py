"""Three-point absolute pose — drop-in for ``visloc.p3p`` (p3p.py:1-306).

``p3p_solve_batch`` runs one GPU thread per minimal sample
(``vl_p3p_solve_batch``): register-resident fp64 resultant quartic, Aberth
root finding, Newton polish, the reference's SVD Procrustes evaluated in
closed form (three points are planar: map the world triangle's plane frame
onto the camera triangle's, then the 2-D Procrustes rotation in that plane;
``csrc/vl_p3p.cuh``), the 1e-8 rad bearing contract and per-sample dedup.  Output order matches the reference: by
sample, then by ascending quartic root.

``sample_minimal_sets`` exposes the device reproduction of numpy's
``Generator.choice(n, 3, replace=False)`` stream that feeds the solver in
``ransac_pnp`` (posest.py:243, :252).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .geometry import Pose, matrix_to_quat

__all__ = ["BEARING_TOL", "p3p_solve", "p3p_solve_batch", "sample_minimal_sets"]

BEARING_TOL = 1e-8


def p3p_solve_batch(bearings, world_points):
    """(R (M,3,3), t (M,3), sample (M,)) for a (B,3,3) batch (p3p.py:57-203)."""
    import torch
    from .posest import _to_device
    f = np.ascontiguousarray(np.asarray(bearings, dtype=np.float64).reshape(-1, 3, 3))
    P = np.ascontiguousarray(np.asarray(world_points, dtype=np.float64).reshape(-1, 3, 3))
    B = f.shape[0]
    if B == 0:
        return np.zeros((0, 3, 3)), np.zeros((0, 3)), np.zeros(0, dtype=np.int64)
    ctx = _lib.context()
    df, dP = _to_device(f), _to_device(P)
    R = torch.empty((4 * B, 3, 3), dtype=torch.float64, device=df.device)
    t = torch.empty((4 * B, 3), dtype=torch.float64, device=df.device)
    idx = torch.empty((4 * B,), dtype=torch.int64, device=df.device)
    m = C.c_int32()
    rc = _lib.lib().vl_p3p_solve_batch(ctx.handle, df.data_ptr(), dP.data_ptr(), B, R.data_ptr(),
                                       t.data_ptr(), idx.data_ptr(), C.byref(m), _lib.stream_ptr())
    ctx.check(rc, "vl_p3p_solve_batch")
    M = m.value
    return R[:M].cpu().numpy(), t[:M].cpu().numpy(), idx[:M].cpu().numpy()


def p3p_solve(bearings, world_points) -> list[Pose]:
    R, t, _ = p3p_solve_batch(np.asarray(bearings, dtype=np.float64)[None],
                              np.asarray(world_points, dtype=np.float64)[None])
    return [Pose(matrix_to_quat(R[i]), t[i]) for i in range(R.shape[0])]


def sample_minimal_sets(seed_or_state, n: int, count: int):
    """``count`` draws of ``choice(n, 3, replace=False)`` generated on the GPU.

    ``seed_or_state`` is an int seed (``default_rng(seed)``) or a numpy
    ``bit_generator.state`` dict.  Returns (samples (count,3) int64, state dict
    after the draws, numpy format).
    """
    import torch
    if isinstance(seed_or_state, dict):
        st = _lib.state_from_numpy(seed_or_state)
    else:
        st = _lib.pcg64_state(int(seed_or_state))
    ctx = _lib.context()
    out = torch.empty((max(count, 1), 3), dtype=torch.int32, device="cuda")
    rc = _lib.lib().vl_sample_minimal_sets(ctx.handle, C.byref(st), int(n), int(count), out.data_ptr(),
                                           _lib.stream_ptr())
    ctx.check(rc, "vl_sample_minimal_sets")
    d = _lib.state_to_dict(st)
    state = {"bit_generator": "PCG64", "state": {"state": d["state"], "inc": d["inc"]},
             "has_uint32": d["has_uint32"], "uinteger": d["uinteger"]}
    return out[:count].cpu().numpy().astype(np.int64), state
