"""CPU checks of the exact solver source the GPU kernels compile.

``libvisloc_hostcheck.so`` is a host-only build of the ``__host__ __device__``
cores (P3P, numpy-compatible sampler, seeding) — a test hook, not a product
path.  Compared against the oracle (itself pinned to the reference).
"""

import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from oracle.p3p import p3p_batch
from oracle.posest import bearings
from oracle.rng import PCG64Stream, sample_batches
from synth_inputs import matches_a

LIB = Path(__file__).resolve().parent.parent / "paper_2601_04185_b200" / "_lib" / "libvisloc_hostcheck.so"
DP = C.POINTER(C.c_double)


@pytest.fixture(scope="module")
def hc():
    if not LIB.exists():
        from paper_2601_04185_b200._build import build
        build()
    L = C.CDLL(str(LIB))
    L.vlh_sample.restype = C.c_uint64
    return L


def _solve(L, f, P):
    R, t = np.zeros(36), np.zeros(12)
    f, P = np.ascontiguousarray(f), np.ascontiguousarray(P)
    m = L.vlh_p3p_solve_one(f.ctypes.data_as(DP), P.ctypes.data_as(DP), R.ctypes.data_as(DP),
                            t.ctypes.data_as(DP))
    return R[:9 * m].reshape(m, 3, 3), t[:3 * m].reshape(m, 3)


def test_p3p_core_matches_reference_golden(hc, golden):
    g = golden("p3p")
    f, P = g["bearings"], g["points"]
    cnt = np.bincount(g["idx"], minlength=f.shape[0])
    ptr, worst = 0, 0.0
    for i in range(f.shape[0]):
        R, t = _solve(hc, f[i], P[i])
        c = cnt[i]
        assert R.shape[0] == c, i
        if c:
            worst = max(worst, np.abs(R - g["R"][ptr:ptr + c]).max(),
                        np.abs(t - g["t"][ptr:ptr + c]).max() / max(1.0, np.abs(g["t"][ptr:ptr + c]).max()))
        ptr += c
    assert worst < 1e-9


def test_p3p_core_degenerate(hc):
    P = np.array([[0, 0, 2.0], [1, 0, 2.0], [2, 0, 2.0]])  # collinear
    f = P / np.linalg.norm(P, axis=1, keepdims=True)
    assert _solve(hc, f, P)[0].shape[0] == 0
    P2 = np.array([[0, 0, 2.0], [0, 0, 2.0], [1, 1, 3.0]])  # coincident
    f2 = P2 / np.linalg.norm(P2, axis=1, keepdims=True)
    assert _solve(hc, f2, P2)[0].shape[0] == 0


def test_p3p_core_random_sweep(hc):
    px, X, w, _ = matches_a(3000, 0.5, 1.0, seed=5)
    b = bearings(px, (700.0, 700.0, 350.0, 350.0))
    rng = np.random.default_rng(9)
    smp = np.stack([rng.choice(3000, 3, replace=False) for _ in range(3000)])
    R, t, idx = p3p_batch(b[smp], X[smp])
    cnt = np.bincount(idx, minlength=3000)
    mism = sum(_solve(hc, b[smp[i]], X[smp[i]])[0].shape[0] != cnt[i] for i in range(3000))
    assert mism == 0


@pytest.mark.parametrize("seed,n", [(0, 3), (1, 4), (2, 7), (3, 2000), (4, 50_000), (5, 200_000),
                                    (2**40 + 1, 10_000), (6, 2**31 - 1)])
def test_sampler_core_bit_exact(hc, seed, n):
    out = np.zeros((2500, 3), dtype=np.int64)
    rej = C.c_int()
    pos = hc.vlh_sample(C.c_uint64(seed), C.c_int64(n), 2500, out.ctypes.data_as(C.POINTER(C.c_int64)),
                        C.byref(rej))
    assert np.array_equal(out, np.array(sample_batches(seed, n, [2500])[0]))
    draws = 4 if n == 3 else 5
    assert pos >= draws * 2500


@pytest.mark.parametrize("seed", [0, 1, 5, 123456789, 2**32 + 5, 2**63 + 7])
def test_seeding_matches_numpy(hc, seed):
    out = np.zeros(4, dtype=np.uint64)
    hc.vlh_seed(C.c_uint64(seed), out.ctypes.data_as(C.POINTER(C.c_uint64)))
    st = np.random.PCG64(seed).state["state"]
    assert (int(out[0]) << 64) | int(out[1]) == st["state"]
    assert (int(out[2]) << 64) | int(out[3]) == st["inc"]


def test_host_chunk_schedule():
    from paper_2601_04185_b200.posest import _host_chunks
    for Q in (1, 2, 5, 16, 17, 100, 1000, 4097):
        ch = _host_chunks(Q)
        assert ch[0][0] == 0 and ch[-1][1] == Q
        assert all(a[1] == b[0] for a, b in zip(ch, ch[1:]))
        assert all(b > a for a, b in ch)
    assert _host_chunks(1000) == [(0, 63), (63, 189), (189, 441), (441, 1000)]
    assert _host_chunks(10, 4) == [(0, 4), (4, 8), (8, 10)]


def test_stage_schedule():
    from paper_2601_04185_b200.posest import _stage_schedule
    for Q in (1, 2, 3, 5, 31, 32, 33, 100, 1000, 4096):
        e = _stage_schedule(Q)
        assert e[-1] == Q and all(b > a for a, b in zip([0] + e, e))
    assert _stage_schedule(1000) == [63, 189, 441, 1000]
