"""GPU engine vs the CPU oracle on the shared parity cases (needs a B200).

Fill order and frontier sets must be bit-exact (per-pixel enter/fill shell
maps encode every shell's frontier set and fill mask), report rows and
counters identical, values within 1e-4 (fp32 colour path).
"""

import math

import numpy as np
import pytest

import cases
from oracle import guidefill_oracle as orc
from paper_1611_05319_b200 import FillParams, Spline, build_guide_field, engine, grid, tracker

pytestmark = pytest.mark.gpu

ALL_CASES = cases.reference_scenes() + cases.random_scenes()
TOL = 1e-4


def _check(case, tracked):
    p = FillParams(**case["params"])
    u, rep, maps = engine._run_fill(case["image"], case["labels"], case["guide"], p,
                                    tracked=tracked, order_log=True)
    ref = orc.fill(case["image"], case["labels"], case["guide"], orc.Params.of(p), tracked=tracked)
    assert np.array_equal(maps["fillshell"], ref["fillshell"]), "fill order differs"
    enter = np.where(ref["enter"] >= 0, ref["enter"], -1)
    assert np.array_equal(maps["enter"], enter), "frontier sets differ"
    assert [tuple(r) for r in rep.rows] == [tuple(r) for r in ref["rows"]]
    assert (rep.iterations, rep.filled, rep.deadlock_fills, rep.unfillable,
            rep.unfillable_count) == (ref["iterations"], ref["filled"], ref["deadlock_fills"],
                                      ref["unfillable"], ref["unfillable_count"])
    err = float(np.abs(u - ref["u"]).max()) if u.size else 0.0
    assert err <= TOL, err


@pytest.mark.parametrize("idx", range(len(ALL_CASES)))
def test_case_tracked(idx):
    _check(ALL_CASES[idx], tracked=True)


@pytest.mark.parametrize("idx", range(len(ALL_CASES)))
def test_case_untracked(idx):
    _check(ALL_CASES[idx], tracked=False)


def test_public_api_matches_oracle():
    case = ALL_CASES[16]  # trk_tracked test_tracker.py:81
    p = FillParams(**case["params"])
    u_t, wm = tracker.run_tracked(case["image"], case["labels"], case["guide"], p, debug=True)
    u_u, rep = engine.inpaint(case["image"], case["labels"], case["guide"], p)
    assert np.array_equal(u_t, u_u)
    assert [r[4] for r in wm.rows] == [r[4] for r in rep.rows]
    assert all(r[3] == 28 * 34 for r in rep.rows)
    assert all(r[3] == r[1] for r in wm.rows)


def test_guide_field_bit_exact():
    for gc in cases.guide_cases():
        spl = [Spline(id=f"s{k}", source="user", direction=s["direction"], points=s["points"],
                      kind=s["kind"]) for k, s in enumerate(gc["splines"])]
        field = build_guide_field(spl, gc["labels"], eta=gc["eta"])
        ref = orc.guide_field([orc.polyline(s["points"], s["kind"]) for s in gc["splines"]],
                              [s["direction"] for s in gc["splines"]], gc["labels"], eta=gc["eta"])
        assert np.array_equal(field, ref)


def test_guide_field_known_answers():
    # test_guide.py:227-282
    labels = np.zeros((30, 40), dtype=np.uint8)
    labels[5:25, 4:36] = 255
    assert not build_guide_field([], labels).any()
    sp = Spline(id="u", source="user", direction=(0.5, 0.5), points=[[0.0, 10.0], [39.0, 10.0]])
    f = build_guide_field([sp], labels)
    assert tuple(f[10, 20]) == (0.5, 0.5)
    assert f[13, 20, 0] == pytest.approx(0.5 * math.exp(-0.5), rel=1e-12)
    assert tuple(f[20, 20]) == (0.0, 0.0)
    assert tuple(f[10, 2]) == (0.0, 0.0)
    a = Spline(id="a", source="user", direction=(1.0, 0.0), points=[[0.0, 8.0], [39.0, 8.0]])
    b = Spline(id="b", source="user", direction=(0.0, 1.0), points=[[0.0, 12.0], [39.0, 12.0]])
    f = build_guide_field([a, b], labels)
    assert f[10, 20, 0] > 0 and f[10, 20, 1] == 0.0
    f = build_guide_field([b, a], labels)
    assert f[10, 20, 1] > 0 and f[10, 20, 0] == 0.0
    bz = Spline(id="bz", source="user", direction=(0.25, 0.0), kind="bezier",
                points=[[0.0, 10.0], [13.0, 10.0], [26.0, 10.0], [39.0, 10.0]])
    assert build_guide_field([bz], labels)[10, 17, 0] == pytest.approx(0.25, rel=1e-12)


def test_confidence_known_answers():
    # test_engine.py:77-139, frozen reference values
    H, W = 12, 31
    lab = np.zeros((H, W), dtype=np.uint8)
    lab[6:, :] = 255
    img = np.zeros((H, W, 1))
    img[:6, :, 0] = 0.8
    th = math.radians(10.0)
    g = (math.cos(th), math.sin(th))
    assert engine.confidence((15, 6), img, lab, (0.0, 1.0), FillParams()) == pytest.approx(0.5, abs=1e-12)
    c = engine.confidence((15, 6), img, lab, g, FillParams())
    assert c == pytest.approx(1.5113912011802175e-61, rel=1e-9)
    assert not engine.ready(c, g, FillParams())
    c = engine.confidence((15, 6), img, lab, g, FillParams(neighborhood="axis_ball"))
    assert c == pytest.approx(4.503504789933916e-24, rel=1e-9)
    v, ok = engine.fill_color((15, 6), img, lab, (0.0, 1.0), FillParams())
    assert ok and v[0] == pytest.approx(0.8, abs=1e-15)
    lab1 = np.full((1, 7), 255, dtype=np.uint8)
    lab1[0, :3] = 0
    img1 = np.zeros((1, 7, 1))
    img1[0, :3, 0] = [0.0, 0.3, 0.9]
    v, ok = engine.fill_color((3, 0), img1, lab1, (1.0, 0.0), FillParams(mu=math.inf))
    assert ok and v[0] == pytest.approx(6.3 / 11.0, rel=1e-14)


def test_sampler_masses_bit_exact():
    # readable / total masses of random points and guides, every radius and mu regime
    rng = np.random.default_rng(2024)
    for r in (1, 2, 3, 4, 5, 6, 7, 9, 12):
        for mu in (0.0, 10.0, 50.0, 100.0, math.inf):
            lab = cases.islands_labels(rng, 30, 60)
            H, W = lab.shape
            img = rng.uniform(size=(H, W, 3))
            p = FillParams(r=r, mu=mu, neighborhood="rotated_ball" if r % 2 else "axis_ball")
            for _ in range(6):
                pt = (int(rng.integers(0, W)), int(rng.integers(0, H)))
                g = tuple(rng.uniform(-1, 1, 2) * (rng.uniform() < 0.8))
                _, rw, tw = engine._point_gather(pt, img, lab, g, p)
                vals, rw0, tw0 = orc.point_sample(img, lab, pt, g, orc.Params.of(p))
                assert rw[0] == rw0[0] and tw[0] == tw0[0], (r, mu, pt, g)
                gv, _, _ = engine._point_gather(pt, img, lab, g, p)
                assert np.abs(gv - vals).max() <= 1e-12


def test_boundaries_match_oracle():
    rng = np.random.default_rng(77)
    for _ in range(10):
        lab = cases.islands_labels(rng, 10, 40)
        for periodic in (False, True):
            assert np.array_equal(grid.active_boundary_mask(lab, periodic),
                                  orc.active_mask(lab, periodic))
            assert grid.inner_boundary(lab, periodic) == {
                (int(i), int(j)) for j, i in zip(*np.nonzero(orc.inner_mask(lab, periodic)))}
            assert grid.outer_boundary(lab, periodic) == {
                (int(i), int(j)) for j, i in zip(*np.nonzero(orc.outer_mask(lab, periodic)))}


def test_bilinear_gather_matches_oracle():
    rng = np.random.default_rng(5)
    lab = cases.islands_labels(rng, 20, 40)
    H, W = lab.shape
    img = rng.uniform(size=(H, W, 2))
    read = lab == 0
    X = rng.uniform(-2, W + 1, 500)
    Y = rng.uniform(-2, H + 1, 500)
    X[:50] = np.round(X[:50])
    Y[:50] = np.round(Y[:50])
    for periodic in (False, True):
        v, ok = grid.bilinear_gather(img, read, X, Y, periodic)
        v0, ok0 = orc.ghost_gather(img, read, X, Y, periodic)
        assert np.array_equal(ok, ok0)
        assert np.abs(v - v0).max() <= 1e-12


def test_spline_guide_extension_equals_field():
    """run_tracked / inpaint accept splines in place of the dense field."""
    from paper_1611_05319_b200 import scenes

    sc = scenes.small_scene(120, 200, band=6, gx=4, gy=3, n_spl=3, seed=21)
    spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
                  kind=s["kind"]) for s in sc.splines]
    p = FillParams(**sc.params)
    field = build_guide_field(spl, sc.labels)
    u1, wm1 = tracker.run_tracked(sc.image, sc.labels, field, p)
    u2, wm2 = tracker.run_tracked(sc.image, sc.labels, spl, p)
    assert np.array_equal(u1, u2) and wm1.rows == wm2.rows
    v1, r1 = engine.inpaint(sc.image, sc.labels, field, p)
    v2, r2 = engine.inpaint(sc.image, sc.labels, spl, p)
    assert np.array_equal(v1, v2) and r1.rows == r2.rows


@pytest.mark.parametrize("bad_at", [(0, 0), (31, 46), (17, 5)])
def test_bad_label_raises_reference_message(bad_at):
    """k_prep flags labels outside {0, 128, 255} (GF_STAT_BAD_LABELS); the API
    raises grid.py:36-46's ValueError with the first bad location."""
    from paper_1611_05319_b200 import tracker

    case = ALL_CASES[0]
    lab = np.array(case["labels"], dtype=np.uint8, copy=True)
    j, i = bad_at
    j, i = min(j, lab.shape[0] - 1), min(i, lab.shape[1] - 1)
    lab[j, i] = 7
    with pytest.raises(ValueError, match="label mask holds value 7"):
        tracker.run_tracked(case["image"], lab, case["guide"], FillParams(**case["params"]))
    with pytest.raises(ValueError, match="label mask holds value 7"):
        engine.inpaint(case["image"], lab, case["guide"], FillParams(**case["params"]))


def test_frame_without_inpaint_pixels():
    case = ALL_CASES[0]
    lab = np.where(case["labels"] == 255, 0, case["labels"]).astype(np.uint8)
    p = FillParams(**case["params"])
    u, rep, maps = engine._run_fill(case["image"], lab, case["guide"], p, tracked=True,
                                    order_log=True)
    ref = orc.fill(case["image"], lab, case["guide"], orc.Params.of(p), tracked=True)
    assert rep.iterations == ref["iterations"] == 0
    assert np.array_equal(u, ref["u"])


def test_fill_loop_seam_replays_recording_hooks():
    """engine._fill_loop (the reference's seam, engine.py:286) with a
    frontier_update hook: one call per shell with the reference's arguments;
    the tracker's own update as the hook reproduces run_tracked; a custom
    rule is refused."""
    case = ALL_CASES[16]  # trk_tracked test_tracker.py:81
    p = FillParams(**case["params"])
    calls = []

    def hook(frontier, fill, filled_idx, lab):
        calls.append((frontier.copy(), fill.copy(), filled_idx.copy()))
        return orc._tracked_update(frontier, fill, filled_idx, lab, p.periodic_x)

    u, lab, rep = engine._fill_loop(case["image"], case["labels"], case["guide"], p, hook)
    u_t, wm = tracker.run_tracked(case["image"], case["labels"], case["guide"], p)
    assert np.array_equal(u, u_t)
    assert rep.rows == wm.rows
    assert len(calls) == rep.iterations
    ref = orc.fill(case["image"], case["labels"], case["guide"], orc.Params.of(p), tracked=True)
    for k, (fr, fm, fi) in enumerate(calls):
        want = np.flatnonzero((ref["enter"].reshape(-1) >= 0) & (ref["enter"].reshape(-1) <= k) &
                              ((ref["fillshell"].reshape(-1) >= k)))
        assert np.array_equal(fr, want) and np.array_equal(fi, fr[fm])
    assert not (lab == 255).any()
    u2, lab2, rep2 = engine._fill_loop(case["image"], case["labels"], case["guide"], p)
    assert np.array_equal(u2, u_t) and all(r[3] == lab2.size for r in rep2.rows)

    def bad_hook(frontier, fill, filled_idx, lab):
        cand, nxt = orc._tracked_update(frontier, fill, filled_idx, lab, p.periodic_x)
        return cand, nxt[1:]

    with pytest.raises(engine.FrontierRuleError):
        engine._fill_loop(case["image"], case["labels"], case["guide"], p, bad_hook)


@pytest.mark.parametrize("seed", range(6))
def test_update_frontier_incremental_equals_rescan(seed):
    """tracker.update_frontier (tracker.py:82-101) on the device: survivors +
    neighbours of the filled pixels, filtered -- equal to a full rescan, for
    index and coordinate-set inputs, fills inside and outside the frontier,
    periodic x (test_tracker.py:23-42)."""
    from paper_1611_05319_b200 import grid as g

    rng = np.random.default_rng(seed)
    lab = cases.islands_labels(rng, 20, 60)
    periodic = bool(seed % 2)
    fr = tracker.FrontierList.from_labels(lab, periodic)
    inp = np.flatnonzero(lab.reshape(-1) == 255)
    pick = rng.choice(inp, size=min(inp.size, int(rng.integers(1, 20))), replace=False)
    lab2 = lab.copy()
    lab2.reshape(-1)[pick] = 0
    want = np.flatnonzero(g.active_boundary_mask(lab2, periodic))
    got = tracker.update_frontier(fr, pick, lab2, periodic)
    assert np.array_equal(got.indices, want) and got.generation == 1
    W = lab.shape[1]
    got2 = tracker.update_frontier(fr, {(int(q % W), int(q // W)) for q in pick}, lab2, periodic)
    assert np.array_equal(got2.indices, want)
