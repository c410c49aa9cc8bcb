"""Depth lifting restated from the reference (numpy, fp64) — TEST INFRASTRUCTURE ONLY.

Follows ``pkg/src/visloc/localizer.py`` (``interp_depth_many`` :87-115,
``lift`` :134-197 without the span checks), ``matchio.filter_matches_arrays``
(:203-218) and ``mapstore.dequantize_depth`` (:122-134).  Inputs are plain
arrays so the GPU box (no reference) can replay golden scenes.
"""

from __future__ import annotations

import math

import numpy as np


def gate(targets, conf, scale_x, scale_y, thr):
    """(src (M,2), tgt (M,2), conf (M,), flat idx (M,)); row-major cells passing the gate."""
    conf = np.asarray(conf)
    keep = (conf >= thr) & (conf > 0)  # NEP 50: python float compared in conf's dtype
    rows, cols = np.nonzero(keep)
    src = np.stack([(cols + 0.5) * scale_x, (rows + 0.5) * scale_y], axis=-1).astype(np.float64)
    tgt = np.asarray(targets)[rows, cols].astype(np.float64)
    return src, tgt, conf[rows, cols].astype(np.float64), rows * conf.shape[1] + cols


def dequantize(codes, d_min, d_max, levels):
    span = math.log(d_max / d_min)
    denom = max(levels - 1, 1)
    c = np.asarray(codes).astype(np.float64)
    d = d_min * np.exp((c - 1.0) / denom * span)
    valid = np.asarray(codes) > 0
    return np.where(valid, d, 0.0).astype(np.float32), valid


def interp(values, valid, pts):
    pts = np.asarray(pts, dtype=np.float64).reshape(-1, 2)
    h, w = valid.shape
    x = pts[:, 0] - 0.5
    y = pts[:, 1] - 0.5
    inside = (x >= 0) & (x <= w - 1) & (y >= 0) & (y <= h - 1)
    x0 = np.clip(np.floor(x), 0, w - 2).astype(np.int64)
    y0 = np.clip(np.floor(y), 0, h - 2).astype(np.int64)
    fx = np.clip(x - x0, 0.0, 1.0)
    fy = np.clip(y - y0, 0.0, 1.0)
    ok = inside & valid[y0, x0] & valid[y0, x0 + 1] & valid[y0 + 1, x0] & valid[y0 + 1, x0 + 1]
    d = values.astype(np.float64)
    v = (d[y0, x0] * (1 - fx) * (1 - fy) + d[y0, x0 + 1] * fx * (1 - fy)
         + d[y0 + 1, x0] * (1 - fx) * fy + d[y0 + 1, x0 + 1] * fx * fy)
    return np.where(ok, v, 0.0), ok


def lift(f_db2q, f_q2db, values, valid, intr_db, db_size, R_db, t_db, thr):
    """(px (M,2), X (M,3), w (M,)) in reference order.

    f_* = (targets, conf, scale_x, scale_y); intr_db = (fx, fy, cx, cy);
    db_size = (W, H) of the database image; R_db, t_db = database pose.
    """
    dh, dw = valid.shape
    sxd, syd = dw / db_size[0], dh / db_size[1]
    fx, fy, cx, cy = intr_db
    Rt = np.asarray(R_db).T
    out_px, out_X, out_w = [], [], []
    src, tgt, conf, _ = gate(*f_db2q, thr)
    if src.shape[0]:
        ix = np.clip((src[:, 0] * sxd).astype(np.int64), 0, dw - 1)
        iy = np.clip((src[:, 1] * syd).astype(np.int64), 0, dh - 1)
        ok = valid[iy, ix]
        d = values.astype(np.float64)[iy, ix]
        xc = np.stack([(src[:, 0] - cx) / fx * d, (src[:, 1] - cy) / fy * d, d], axis=-1)
        Xw = (xc - t_db) @ Rt.T
        out_px.append(tgt[ok])
        out_X.append(Xw[ok])
        out_w.append(conf[ok])
    src, tgt, conf, _ = gate(*f_q2db, thr)
    if src.shape[0]:
        d, ok = interp(values, valid, tgt * np.array([sxd, syd]))
        xc = np.stack([(tgt[:, 0] - cx) / fx * d, (tgt[:, 1] - cy) / fy * d, d], axis=-1)
        Xw = (xc - t_db) @ Rt.T
        out_px.append(src[ok])
        out_X.append(Xw[ok])
        out_w.append(conf[ok])
    if not out_px:
        return np.zeros((0, 2)), np.zeros((0, 3)), np.zeros(0)
    return np.concatenate(out_px), np.concatenate(out_X), np.concatenate(out_w)
