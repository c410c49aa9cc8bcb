"""Pose / quaternion algebra restated from the reference (fp64, numpy).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

A pose is the pair ``(q, t)``: scalar-first unit quaternion canonicalised to
w >= 0 and translation, camera-from-world (``X_cam = R X_world + t``).
References: ``pkg/src/visloc/geometry.py`` — ``quat_multiply`` :79-89,
``quat_to_matrix`` :92-100, ``matrix_to_quat`` (Shepperd) :103-127,
``rotvec_to_quat`` :130-141, ``Pose.__post_init__`` :160-171,
``pose_error`` :268-273.
"""

from __future__ import annotations

import math

import numpy as np


def canon(q: np.ndarray) -> np.ndarray:
    """Normalisation rule of ``Pose.__post_init__`` (geometry.py:160-171)."""
    q = np.asarray(q, dtype=np.float64).reshape(4)
    n = np.linalg.norm(q)
    if abs(n - 1.0) > 1e-6:
        raise ValueError(f"quaternion norm {n} too far from 1")
    if abs(n - 1.0) > 1e-12:
        q = q / n
    if q[0] < 0:
        q = -q
    return q


def qmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array([
        aw * bw - ax * bx - ay * by - az * bz,
        aw * bx + ax * bw + ay * bz - az * by,
        aw * by - ax * bz + ay * bw + az * bx,
        aw * bz + ax * by - ay * bx + az * bw,
    ])


def q2R(q: np.ndarray) -> np.ndarray:
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def R2q(R: np.ndarray) -> np.ndarray:
    """Shepperd's method, branch order of geometry.py:103-127, then unit-normalised."""
    R = np.asarray(R, dtype=np.float64)
    d0, d1, d2 = R[0, 0], R[1, 1], R[2, 2]
    tr = d0 + d1 + d2
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2.0
        q = [0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s]
    elif d0 >= d1 and d0 >= d2:
        s = math.sqrt(1.0 + d0 - d1 - d2) * 2.0
        q = [(R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s, (R[0, 2] + R[2, 0]) / s]
    elif d1 >= d2:
        s = math.sqrt(1.0 + d1 - d0 - d2) * 2.0
        q = [(R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s, (R[1, 2] + R[2, 1]) / s]
    else:
        s = math.sqrt(1.0 + d2 - d0 - d1) * 2.0
        q = [(R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s, (R[1, 2] + R[2, 1]) / s, 0.25 * s]
    q = np.array(q)
    return q / np.linalg.norm(q)


def rotvec2q(w: np.ndarray) -> np.ndarray:
    w = np.asarray(w, dtype=np.float64)
    th = np.linalg.norm(w)
    if th < 1e-12:
        h = 0.5 * th
        q = np.array([1.0 - h * h / 2.0, 0.5 * w[0], 0.5 * w[1], 0.5 * w[2]])
        return q / np.linalg.norm(q)
    ax = w / th
    s = math.sin(0.5 * th)
    return np.array([math.cos(0.5 * th), ax[0] * s, ax[1] * s, ax[2] * s])


def pose_from_Rt(R, t):
    """``Pose.from_rt`` (geometry.py:174-176): quaternion round trip."""
    return canon(R2q(R)), np.asarray(t, dtype=np.float64).reshape(3).copy()


def apply_delta(pose, delta):
    """Left composition ``refine.apply_delta`` (refine.py:80-87)."""
    q, t = pose
    dq = rotvec2q(np.asarray(delta[:3], dtype=np.float64))
    qn = qmul(dq, q)
    Rd = q2R(canon(dq))
    return canon(qn), Rd @ t + np.asarray(delta[3:6], dtype=np.float64)


def rot_err_deg(qa, qb) -> float:
    qr = qmul(qa, np.array([qb[0], -qb[1], -qb[2], -qb[3]]))
    return math.degrees(2.0 * math.atan2(np.linalg.norm(qr[1:]), abs(qr[0])))


def center(pose) -> np.ndarray:
    q, t = pose
    return -(q2R(q).T @ t)


def pose_err(a, b) -> tuple[float, float]:
    """(rotation deg, camera-centre distance m) as ``pose_error`` (geometry.py:268-273)."""
    return rot_err_deg(a[0], b[0]), float(np.linalg.norm(center(a) - center(b)))
