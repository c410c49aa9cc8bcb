"""Depth-map codecs restated from the reference (numpy, fp64) — TEST INFRASTRUCTURE ONLY.

Follows ``pkg/src/visloc/mapstore.py``: ``quantize_depth`` :96-119 (log
quantisation, round half away from zero), ``dequantize_depth`` :122-134,
``_downsample_codes_nearest_valid`` :390-414 (valid code nearest the block
centre, first row-major on ties) and ``_requantize_codes`` :417-425.
Pinned bit for bit against ``tests/golden/mapstore.npz`` (made by the real
reference, ``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import math

import numpy as np


def quantize(values, valid, d_min=0.25, d_max=128.0, levels=255):
    """f32 depth + valid -> codes (u8 for levels <= 255 else u16), mapstore.py:112-119."""
    vals = np.asarray(values).astype(np.float32).astype(np.float64)
    span = math.log(d_max) - math.log(d_min)
    with np.errstate(divide="ignore", invalid="ignore"):
        u = (np.log(np.clip(vals, d_min, d_max)) - math.log(d_min)) / span
    codes = 1 + np.floor(u * (levels - 1) + 0.5)
    codes = np.where(np.asarray(valid, dtype=bool), codes, 0)
    return codes.astype(np.uint8 if levels <= 255 else np.uint16)


def downsample_nearest_valid(codes, factor):
    """Per block keep the valid code nearest the centre (mapstore.py:390-414)."""
    codes = np.asarray(codes)
    if factor == 1:
        return codes.copy()
    h, w = codes.shape
    oh, ow = (h + factor - 1) // factor, (w + factor - 1) // factor
    out = np.zeros((oh, ow), dtype=codes.dtype)
    for br in range(oh):
        r0, r1 = br * factor, min((br + 1) * factor, h)
        for bc in range(ow):
            c0, c1 = bc * factor, min((bc + 1) * factor, w)
            block = codes[r0:r1, c0:c1]
            rows, cols = np.nonzero(block > 0)
            if rows.size == 0:
                continue
            d2 = (rows - (r1 - r0 - 1) / 2.0) ** 2 + (cols - (c1 - c0 - 1) / 2.0) ** 2
            best = int(np.argmin(d2))
            out[br, bc] = block[rows[best], cols[best]]
    return out


def requantize(codes, levels, new_levels):
    """Level-count change of codes (mapstore.py:417-425)."""
    codes = np.asarray(codes)
    if new_levels == levels:
        return codes.copy()
    u = (codes.astype(np.float64) - 1.0) / max(levels - 1, 1)
    out = 1 + np.floor(u * (new_levels - 1) + 0.5)
    out = np.where(codes > 0, out, 0)
    return out.astype(np.uint8 if new_levels <= 255 else np.uint16)
