"""The C-ABI library loads on CPU and exports every symbol include/*.h declares."""

import ctypes as C
import re
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        txt = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(vl_\w+)\s*\(", txt, flags=re.M))
    return names


def test_library_exports_declared_symbols():
    from paper_2601_04185_b200 import _lib
    L = _lib.lib()
    decl = _declared()
    assert decl, "no declarations parsed"
    assert decl == set(_lib.EXPORTED_SYMBOLS)
    for name in decl:
        assert hasattr(L, name), name


def test_seed_helper_matches_numpy():
    from paper_2601_04185_b200 import _lib
    for seed in (0, 7, 2**40 + 11):
        st = _lib.state_to_dict(_lib.pcg64_state(seed))
        ref = np.random.PCG64(seed).state
        assert st["state"] == ref["state"]["state"] and st["inc"] == ref["state"]["inc"]


def test_no_device_fails_loudly():
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_04185_b200 import RansacConfig, ransac_pnp
    from paper_2601_04185_b200._lib import VislocError
    from synth_inputs import INTR_A, matches_a
    px, X, w, _ = matches_a(50)
    with pytest.raises(VislocError):
        ransac_pnp((px, X, w), INTR_A, RansacConfig(seed=0))
