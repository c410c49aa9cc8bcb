"""Recall / median bookkeeping (localizer.evaluate, reference localizer.py:263-305),
checked on the cases the reference's test_localizer.py:208-280 covers."""

import math

import numpy as np
import pytest

from paper_2601_04185_b200.geometry import Pose, rotvec_to_quat
from paper_2601_04185_b200.localizer import EvalThresholds, evaluate
from paper_2601_04185_b200.posest import PoseEstimate


def _est(ok=True):
    return PoseEstimate(pose=Pose.identity(), inlier_count=10 if ok else 0, inlier_flags=np.zeros(0, bool),
                        score=0.0 if ok else math.inf, iterations=1, converged=ok)


def _gt(trans, rot_deg):
    return Pose(rotvec_to_quat(np.array([0.0, 0.0, math.radians(rot_deg)])), np.array([trans, 0.0, 0.0]))


def test_hand_counted_recalls():
    res = evaluate([(_est(), _gt(0.1, 1.0)), (_est(), _gt(0.7, 3.0))], EvalThresholds())
    assert res.recalls == [0.5, 0.5, 1.0]


def test_all_exact_and_all_failed():
    res = evaluate([(_est(), Pose.identity())] * 4, EvalThresholds())
    assert res.recalls == [1.0, 1.0, 1.0] and res.median_translation_m == 0.0 and res.median_rotation_deg < 1e-12
    res = evaluate([(_est(False), Pose.identity())] * 3, EvalThresholds())
    assert res.recalls == [0.0, 0.0, 0.0] and math.isnan(res.median_translation_m) and res.num_failed == 3


def test_medians_lower_and_skip_failures():
    res = evaluate([(_est(), _gt(0.2, 0.5)), (_est(False), Pose.identity()), (_est(), _gt(0.4, 1.5))],
                   EvalThresholds())
    assert res.median_translation_m == pytest.approx(0.2) and res.num_queries == 3
    res = evaluate([(_est(), _gt(t, 0.1)) for t in (0.1, 0.2, 0.3, 0.4)], EvalThresholds())
    assert res.median_translation_m == pytest.approx(0.2)


def test_recall_monotone_and_errors():
    rng = np.random.default_rng(0)
    pairs = [(_est(), _gt(float(rng.uniform(0, 1.5)), float(rng.uniform(0, 12)))) for _ in range(40)]
    grid = [(t, r) for t in (0.1, 0.3, 0.6, 1.2) for r in (1.0, 4.0, 11.0)]
    by = dict(zip(grid, evaluate(pairs, EvalThresholds(tuple(grid))).recalls))
    for a in grid:
        for b in grid:
            if a[0] <= b[0] and a[1] <= b[1]:
                assert by[a] <= by[b]
    with pytest.raises(ValueError):
        evaluate([], EvalThresholds())
    with pytest.raises(ValueError):
        EvalThresholds(((0.0, 1.0),))
    assert EvalThresholds.parse("0.25:2,0.5:5,1:10").pairs == ((0.25, 2.0), (0.5, 5.0), (1.0, 10.0))
