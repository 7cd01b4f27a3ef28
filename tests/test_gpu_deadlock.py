"""Deadlock-heavy regime on the GPU (SURVEY.md section 7 hard part 2, Appendix B).

256x256 half-planes with a rotated guide at 10/25/40/73 degrees under smart
order, mu 50 / 100: 4,288-22,058 shells, most of them filling one pixel
through the deadlock guard (engine.py:334-348: argmax confidence, first
index on ties).  Checked against the reference's own outputs
(tests/golden/deadlock_golden.npz, made by
tests/golden/make_deadlock_golden.py): per-pixel enter / fill shells
bit-exact, every report row identical, values within 1e-4.
"""

import os

import numpy as np
import pytest

import cases
from paper_1611_05319_b200 import FillParams, engine

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "deadlock_golden.npz")
DL_CASES = cases.deadlock_scenes()
TOL = 1e-4


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("idx", range(len(DL_CASES)))
def test_deadlock_chain_parity(gold, idx):
    case = DL_CASES[idx]
    key = f"d{idx:03d}"
    assert str(gold[f"{key}_name"]) == case["name"]
    p = FillParams(**case["params"])
    u, rep, maps = engine._run_fill(case["image"], case["labels"], case["guide"], p,
                                    tracked=True, order_log=True)
    stats = [rep.iterations, rep.filled, rep.deadlock_fills, int(rep.unfillable),
             rep.unfillable_count]
    assert stats == gold[f"{key}_stats"].tolist()
    rows = np.array([(r[1], r[4]) for r in rep.rows], dtype=np.int32).reshape(-1, 2)
    assert np.array_equal(rows, gold[f"{key}_rows"])
    assert np.array_equal(maps["fillshell"], gold[f"{key}_fillshell"]), "fill order differs"
    assert np.array_equal(maps["enter"], gold[f"{key}_enter"]), "frontier sets differ"
    inp = case["labels"] == 255
    assert np.array_equal(u[~inp], case["image"][~inp])
    err = float(np.abs(u[inp] - gold[f"{key}_uq"] / 65535.0).max())
    assert err <= TOL + 1e-5, err  # + the fixture's 16-bit quantisation


@pytest.mark.parametrize("idx", [2, 6])
def test_deadlock_chain_untracked_equals_tracked(gold, idx):
    case = DL_CASES[idx]
    key = f"d{idx:03d}"
    p = FillParams(**case["params"])
    u, rep, maps = engine._run_fill(case["image"], case["labels"], case["guide"], p,
                                    tracked=False, order_log=True)
    assert np.array_equal(maps["fillshell"], gold[f"{key}_fillshell"])
    assert rep.deadlock_fills == int(gold[f"{key}_stats"][2])
