"""Parity bars shared by the GPU tests (BASELINE.json north_star).

* inlier masks bit-exact except points whose reprojection error lies within
  1e-6 px of tau under the compared pose (checked both ways: against the
  reference's mask and against the reference msac_score of the GPU pose);
* final pose within 0.01 deg rotation and 1e-4 relative translation.
"""

from __future__ import annotations

import numpy as np

from oracle import geometry as og
from oracle.posest import errors_sq


def near_threshold(q, t, px, X, intr, tau, tol=1e-6):
    """Points whose reprojection error under pose (q, t) is within `tol` px of tau."""
    e = np.sqrt(errors_sq(og.q2R(q), t, X, px, intr))
    return np.abs(e - tau) < tol


def check_mask(flags, ref_flags, q, t, px, X, intr, tau, tol=1e-6, q_ref=None, t_ref=None):
    """Mask differences are allowed only at points within `tol` px of tau under
    the GPU pose (q, t) or the reference pose (q_ref, t_ref)."""
    flags, ref_flags = np.asarray(flags, bool), np.asarray(ref_flags, bool)
    assert flags.shape == ref_flags.shape, (flags.shape, ref_flags.shape)
    diff = flags != ref_flags
    if not diff.any():
        return 0
    amb = near_threshold(q, t, px, X, intr, tau, tol)
    if q_ref is not None:
        amb |= near_threshold(q_ref, t_ref, px, X, intr, tau, tol)
    bad = diff & ~amb
    assert not bad.any(), f"{int(bad.sum())} mask differences away from tau (of {int(diff.sum())})"
    return int(diff.sum())


def check_pose(q, t, q_ref, t_ref, rot_deg=0.01, rel_t=1e-4):
    rot = og.rot_err_deg(q, q_ref)
    assert rot < rot_deg, rot
    rel = np.linalg.norm(np.asarray(t) - t_ref) / max(np.linalg.norm(t_ref), 1e-12)
    assert rel < rel_t, rel
    return rot, rel
