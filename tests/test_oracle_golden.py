"""The CPU oracle reproduces the reference's own outputs bit for bit.

Fixtures come from tests/golden/make_golden.py, which runs the reference
package (/root/reference) itself.  This pins the oracle before it is used
to check the CUDA engine.
"""

import os

import numpy as np
import pytest

import cases
from oracle import guidefill_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ALL_CASES = cases.reference_scenes() + cases.random_scenes()


@pytest.fixture(scope="module")
def fill_gold():
    return np.load(os.path.join(GOLD, "fill_golden.npz"))


@pytest.mark.parametrize("idx", range(len(ALL_CASES)))
def test_fill_matches_reference(fill_gold, idx):
    case = ALL_CASES[idx]
    key = f"c{idx:03d}"
    assert str(fill_gold[f"{key}_name"]) == case["name"]
    res = orc.fill(case["image"], case["labels"], case["guide"], orc.Params(**case["params"]),
                   tracked=case["tracked"])
    assert res["u"].tobytes() == fill_gold[f"{key}_u"].tobytes()
    rows = np.array(res["rows"], dtype=np.int64).reshape(-1, 5)
    assert np.array_equal(rows, fill_gold[f"{key}_rows"])
    stats = [res["iterations"], res["filled"], res["deadlock_fills"], int(res["unfillable"]),
             res["unfillable_count"]]
    assert stats == fill_gold[f"{key}_stats"].tolist()
    assert np.array_equal(res["enter"], fill_gold[f"{key}_enter"])
    assert np.array_equal(res["fillshell"], fill_gold[f"{key}_fillshell"])


def test_guide_field_matches_reference():
    gold = np.load(os.path.join(GOLD, "guide_golden.npz"))
    for idx, gc in enumerate(cases.guide_cases()):
        key = f"g{idx:03d}"
        polys = [orc.polyline(s["points"], s["kind"]) for s in gc["splines"]]
        for k, p in enumerate(polys):
            assert p.tobytes() == gold[f"{key}_poly{k}"].tobytes()
        field = orc.guide_field(polys, [s["direction"] for s in gc["splines"]], gc["labels"],
                                eta=gc["eta"])
        assert field.tobytes() == gold[f"{key}_field"].tobytes()


def test_known_answers():
    kat = np.load(os.path.join(GOLD, "kat_golden.npz"))
    H, W = 12, 31
    lab = np.zeros((H, W), dtype=np.uint8)
    lab[6:, :] = 255
    img = np.zeros((H, W, 1))
    img[:6, :, 0] = 0.8
    import math
    th = math.radians(10.0)
    g10 = (math.cos(th), math.sin(th))
    _, rw, tw = orc.point_sample(img, lab, (15, 6), (0.0, 1.0), orc.Params())
    assert rw[0] / tw[0] == float(kat["conf_flat"]) == 0.5
    _, rw, tw = orc.point_sample(img, lab, (15, 6), g10, orc.Params())
    assert rw[0] / tw[0] == float(kat["conf_rot10"])
    assert rw[0] / tw[0] == pytest.approx(1.5113912011802175e-61, rel=1e-9)
    _, rw, tw = orc.point_sample(img, lab, (15, 6), g10, orc.Params(neighborhood="axis_ball"))
    assert rw[0] / tw[0] == pytest.approx(4.503504789933916e-24, rel=1e-9)
    lab1 = np.full((1, 7), 255, dtype=np.uint8)
    lab1[0, :3] = 0
    img1 = np.zeros((1, 7, 1))
    img1[0, :3, 0] = [0.0, 0.3, 0.9]
    v, _, _ = orc.point_sample(img1, lab1, (3, 0), (1.0, 0.0), orc.Params(mu=math.inf))
    assert v[0, 0] == float(kat["fill_muinf"])


def test_disk_sizes():
    # test_grid.py:185-190 disk cardinalities 5/13/29
    assert [len(orc.disk_offsets(r)) for r in (1, 2, 3)] == [5, 13, 29]


CT_CASES = cases.coherence_scenes()


@pytest.mark.parametrize("idx", range(len(CT_CASES)))
def test_coherence_fill_matches_reference(idx):
    """g_source = modified_structure_tensor (engine.py:243-249, guide.py:330-355)."""
    gold = np.load(os.path.join(GOLD, "coherence_golden.npz"))
    case = CT_CASES[idx]
    key = f"c{idx:03d}"
    assert str(gold[f"{key}_name"]) == case["name"]
    res = orc.fill(case["image"], case["labels"], case["guide"], orc.Params(**case["params"]),
                   tracked=case["tracked"])
    assert res["u"].tobytes() == gold[f"{key}_u"].tobytes()
    assert np.array_equal(np.array(res["rows"], dtype=np.int64).reshape(-1, 5), gold[f"{key}_rows"])
    assert np.array_equal(res["enter"], gold[f"{key}_enter"])
    assert np.array_equal(res["fillshell"], gold[f"{key}_fillshell"])


def test_coherence_directions_match_reference():
    gold = np.load(os.path.join(GOLD, "coherence_golden.npz"))
    img, lab = cases.edge_block()
    for s, r in ((2.0, 4.0), (1.0, 2.0)):
        g = orc.coherence_directions(img, lab == 0, gold["dirs_ii"], gold["dirs_jj"], sigma=s, rho=r)
        assert g.tobytes() == gold[f"dirs_s{s:g}_r{r:g}"].tobytes()


DL_CASES = cases.deadlock_scenes(thetas=(73.0,), mus=(50.0,))


def test_oracle_deadlock_chain_matches_reference():
    """The oracle in the deadlock regime: the 73 degree
    half-plane, 4,288 shells, bit-exact against the reference's fixture (the
    other angles take minutes on the CPU and are checked on the GPU only)."""
    gold = np.load(os.path.join(GOLD, "deadlock_golden.npz"))
    case = DL_CASES[0]
    key = "d006"
    assert str(gold[f"{key}_name"]) == case["name"]
    res = orc.fill(case["image"], case["labels"], case["guide"],
                   orc.Params(**case["params"]), tracked=True)
    assert np.array_equal(res["fillshell"], gold[f"{key}_fillshell"])
    assert np.array_equal(res["enter"], gold[f"{key}_enter"])
    rows = np.array([(r[1], r[4]) for r in res["rows"]], dtype=np.int32).reshape(-1, 2)
    assert np.array_equal(rows, gold[f"{key}_rows"])
    inp = case["labels"] == 255
    assert float(np.abs(res["u"][inp] - gold[f"{key}_uq"] / 65535.0).max()) <= 1e-5
