"""Automatic spline detection: the CPU oracle (oracle/detect_oracle.py) pinned.

* ring, tensors, make_spline and the seed clustering against the reference's
  own outputs (tests/golden/detect_golden.npz, made by
  tests/golden/make_detect_golden.py from /root/reference) -- bit for bit;
* the Canny step (scikit-image, absent here: parity unpinned) against the
  reference's detection tests (test_guide.py:154-216), restated.
"""

import math
import os

import numpy as np
import pytest

import cases
from oracle import detect_oracle as det

GOLD = os.path.join(os.path.dirname(__file__), "golden", "detect_golden.npz")
SCENES = cases.detect_scenes()


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("s", range(len(SCENES)))
def test_oracle_ring_tensors_splines_match_reference(gold, s):
    name, img, lab = SCENES[s]
    key = f"s{s:02d}"
    assert str(gold[f"{key}_name"]) == name
    ring = sorted(det.compute_ring(lab), key=lambda p: (p[1], p[0]))
    assert np.array_equal(np.array(ring).reshape(-1, 2), gold[f"{key}_ring"])
    for k, (i, j) in enumerate(gold[f"{key}_pick"]):
        assert np.array_equal(det.structure_tensor(img, (i, j)), gold[f"{key}_tensor"][k])
        sp = det.make_spline((i, j), img, lab)
        ref = gold[f"{key}_spline"][k]
        if sp is None:
            assert np.isnan(ref[0])
        else:
            got = np.concatenate([sp[0], sp[1], np.array(sp[2])])
            assert np.array_equal(got, ref)


def test_oracle_clustering_matches_reference(gold):
    hits = [(int(a), int(b), float(c)) for a, b, c in gold["hits"]]
    assert np.array_equal(np.array(det.cluster_seeds(hits)), gold["clustered"])


def test_canny_restatement_meets_reference_detection_tests():
    """test_guide.py:154-216 on the oracle (scikit-image's canny restated)."""
    (_, hp, hp_lab), (_, blk, blk_lab), (_, par, par_lab) = SCENES[:3]
    assert det.detect_edge_seeds(np.full(blk.shape, 0.5), blk_lab) == []
    seeds = det.detect_edge_seeds(blk, blk_lab)
    assert {(i, j) for i, j, _ in seeds} == {(30, 11), (30, 48)}
    assert all(s > 0.05 for _, _, s in seeds)
    spl = det.detect_splines(blk, blk_lab)
    assert len(spl) == 2
    for start, end, d in spl:
        assert abs(d[0]) < 0.05 and abs(abs(d[1]) - 1.0) < 1e-3 and math.hypot(*d) <= 1.0
    top = next(sp for sp in spl if sp[0][1] < 30)
    assert top[2][1] > 0 and top[1][1] >= 34.5
    spl = det.detect_splines(hp, hp_lab)
    assert len(spl) == 1
    assert abs(math.degrees(math.atan2(spl[0][2][1], spl[0][2][0])) - 45.0) < 2.0
    assert spl[0][1][1] > 95.0
    assert det.make_spline((50, 37), par, par_lab) is None
    assert det.detect_splines(par, par_lab) == []
