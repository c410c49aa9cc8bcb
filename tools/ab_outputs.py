"""Dump estimator outputs for an A/B bit-identity check between two library builds.

    VISLOC_B200_LIB=<lib> python tools/ab_outputs.py OUT.npz [queries] [n]
    python tools/ab_outputs.py --compare A.npz B.npz
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]


def dump(out, Q=200, n=20000):
    import torch
    from bench import query_a, query_seed
    from paper_2601_04185_b200.geometry import CameraIntrinsics
    from paper_2601_04185_b200.posest import RansacConfig, ransac_pnp_device
    res = {}
    for tag, outl, mi, eta, seed0 in (("fixed", 0.7, 3000, 1e-300, 3000), ("low", 0.95, 20000, 1e-4, 4000),
                                      ("one", 0.6, 5000, 1e-300, 5000)):
        q = 1 if tag == "one" else Q
        qs = [query_a(i, n, outl, 1.0, seed0) for i in range(q)]
        px = torch.from_numpy(np.concatenate([a[0] for a in qs])).cuda()
        X = torch.from_numpy(np.concatenate([a[1] for a in qs])).cuda()
        w = torch.from_numpy(np.concatenate([a[2] for a in qs])).cuda()
        off = np.arange(q + 1, dtype=np.int64) * n
        intr = [CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)] * q
        o = ransac_pnp_device(px, X, w, off, intr, [query_seed(i, seed0) for i in range(q)],
                              RansacConfig(max_iterations=mi, miss_probability=eta))
        for k, v in o.items():
            res[f"{tag}_{k}"] = v.cpu().numpy()
    np.savez(out, **res)


def compare(a, b):
    A, B = np.load(a), np.load(b)
    bad = [k for k in A.files if not np.array_equal(A[k], B[k])]
    for k in bad:
        d = np.abs(A[k].astype(np.float64) - B[k].astype(np.float64)).max()
        print(f"DIFF {k}: max |a-b| {d:.3e}")
    print("identical" if not bad else f"{len(bad)} arrays differ")


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        compare(sys.argv[2], sys.argv[3])
    else:
        dump(sys.argv[1], *(int(x) for x in sys.argv[2:]))
