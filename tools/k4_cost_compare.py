"""fp32 ranking costs of the library's k_score vs the reference's own (tools only).

    [VISLOC_B200_LIB=<variant.so>] python tools/k4_cost_compare.py

Scores the reference's 600 golden hypotheses (tests/golden/score.npz, written
by `_score_hypotheses`, posest.py:178-220) through `vl_score_hypotheses` and
prints the relative error statistics — used to compare k_score variants (e.g.
the IEEE-division build) against the reference's numbers.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]


def main():
    import paper_2601_04185_b200 as vl
    from paper_2601_04185_b200.posest import score_hypotheses
    g = np.load(ROOT / "tests" / "golden" / "score.npz")
    intr = vl.CameraIntrinsics(700.0, 700.0, 350.0, 350.0, 700, 700)
    got = score_hypotheses(g["R"], g["t"], g["X"], g["px"], g["w"], intr, float(g["tau"]))
    rel = np.abs(got - g["costs"]) / np.abs(g["costs"])
    print(f"max rel {rel.max():.3e} median {np.median(rel):.3e} exact {int((got == g['costs']).sum())}/{got.size}")


if __name__ == "__main__":
    main()
