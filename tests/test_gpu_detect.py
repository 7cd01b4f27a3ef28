"""Automatic spline detection on the GPU (guide.detect_splines: gf_detect_edges,
gf_structure_eigen, gf_trace_rays).

Against the reference's own outputs where they need no Canny
(tests/golden/detect_golden.npz: ring, tensors, make_spline), against the CPU
oracle for the whole pipeline (oracle/detect_oracle.py, whose Canny
restatement is unpinned -- scikit-image is absent), and against the
reference's detection tests (test_guide.py:55-216) directly.
"""

import math
import os

import numpy as np
import pytest

import cases
from oracle import detect_oracle as det
from paper_1611_05319_b200 import guide

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "detect_golden.npz")
SCENES = cases.detect_scenes()


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("s", range(len(SCENES)))
def test_ring_tensor_rays_match_reference(gold, s):
    name, img, lab = SCENES[s]
    key = f"s{s:02d}"
    ring = sorted(guide.compute_ring(lab), key=lambda p: (p[1], p[0]))
    assert np.array_equal(np.array(ring).reshape(-1, 2), gold[f"{key}_ring"])
    for k, (i, j) in enumerate(gold[f"{key}_pick"]):
        J = guide.structure_tensor(img, (i, j))
        assert np.array_equal(J, gold[f"{key}_tensor"][k])  # the reference's bits
        ref_m = gold[f"{key}_mtensor"][k]
        if np.isnan(ref_m[0, 0]):
            with pytest.raises(guide.ZeroMassError):
                guide.modified_structure_tensor(img, lab, (i, j))
        else:
            assert np.array_equal(guide.modified_structure_tensor(img, lab, (i, j)), ref_m)
        sp = guide.make_spline((i, j), img, lab)
        ref = gold[f"{key}_spline"][k]
        if np.isnan(ref[0]):
            assert sp is None
        else:
            got = np.concatenate([sp.points.reshape(-1), np.array(sp.direction)])
            assert np.array_equal(got, ref), (got, ref)


@pytest.mark.parametrize("s", range(len(SCENES)))
def test_detection_matches_oracle(s):
    name, img, lab = SCENES[s]
    hits = det.detect_hits(img, lab)
    seeds = guide.detect_edge_seeds(img, lab)
    assert [(i, j) for i, j, _ in seeds] == [(i, j) for i, j, _ in det.cluster_seeds(hits)]
    for (_, _, a), (_, _, b) in zip(seeds, det.cluster_seeds(hits)):
        assert a == b  # the same ops on the same doubles
    got = guide.detect_splines(img, lab)
    want = det.detect_splines(img, lab)
    assert len(got) == len(want)
    for k, (sp, (start, end, d)) in enumerate(zip(got, want)):
        assert sp.id == f"auto-{k}" and sp.source == "auto"
        # bit for bit: numpy's transcendentals on the device, math.tanh on the host
        assert np.array_equal(np.asarray(sp.points), np.stack([start, end]))
        assert tuple(sp.direction) == tuple(d)


def test_reference_detection_tests():
    """test_guide.py:55-216, on the device path."""
    (_, hp, hp_lab), (_, blk, blk_lab), (_, par, par_lab) = SCENES[:3]
    assert guide.compute_ring(hp_lab) == {(i, 37) for i in range(100)}
    assert guide.ring_distance() == 13
    small = np.zeros((20, 20), dtype=np.uint8)
    small[8:12, 8:12] = 255
    with pytest.raises(guide.EmptyRingError):
        guide.compute_ring(small)
    with pytest.raises(guide.EmptyRingError):
        guide.compute_ring(np.zeros((40, 40), dtype=np.uint8))
    guide.structure_tensor(hp, (37, 37), labels=hp_lab)
    with pytest.raises(guide.WindowOverlapError):
        guide.structure_tensor(hp, (37, 38), labels=hp_lab)
    with pytest.raises(guide.ZeroMassError):
        guide.modified_structure_tensor(hp, hp_lab, (50, 70))
    ring_deg = math.degrees(guide.tensor_orientation(guide.structure_tensor(hp, (37, 37))))
    assert abs(ring_deg - 45.0) < 2.0
    mst_deg = math.degrees(guide.tensor_orientation(
        guide.modified_structure_tensor(hp, hp_lab, (50, 50))))
    assert mst_deg == pytest.approx(57.19707071708637, abs=1e-9)
    assert guide.detect_edge_seeds(np.full(blk.shape, 0.5), blk_lab) == []
    seeds = guide.detect_edge_seeds(blk, blk_lab)
    assert {(i, j) for i, j, _ in seeds} == {(30, 11), (30, 48)}
    spl = guide.detect_splines(blk, blk_lab)
    assert [sp.id for sp in spl] == ["auto-0", "auto-1"]
    for sp in spl:
        assert abs(sp.direction[0]) < 0.05 and abs(abs(sp.direction[1]) - 1.0) < 1e-3
    top = next(sp for sp in spl if sp.points[0, 1] < 30)
    assert top.direction[1] > 0 and top.points[1, 1] >= 34.5
    spl = guide.detect_splines(hp, hp_lab)
    assert len(spl) == 1 and spl[0].points[1, 1] > 95.0
    assert abs(math.degrees(math.atan2(spl[0].direction[1], spl[0].direction[0])) - 45.0) < 2.0
    assert guide.make_spline((50, 37), par, par_lab) is None
    assert guide.detect_splines(par, par_lab) == []


def test_detected_splines_drive_the_fill():
    """A disocclusion frame filled with its detected splines: the same fill as
    the oracle with the oracle's splines (guide field and order bit-exact)."""
    from oracle import guidefill_oracle as orc
    from paper_1611_05319_b200 import FillParams, build_guide_field, scenes, tracker

    sc = scenes.small_scene(180, 240, band=8, gx=3, gy=2, n_spl=2, seed=11)
    spl = guide.detect_splines(sc.image, sc.labels)
    want = det.detect_splines(sc.image, sc.labels)
    assert len(spl) == len(want)
    field = build_guide_field(spl, sc.labels)
    p = FillParams(**sc.params)
    u, wm = tracker.run_tracked(sc.image, sc.labels, field, p)
    ref = orc.fill(sc.image, sc.labels, field, orc.Params.of(p), tracked=True)
    assert [r[4] for r in wm.rows] == [r[4] for r in ref["rows"]]
    assert float(np.abs(u - ref["u"]).max()) <= 1e-4
