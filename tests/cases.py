"""Deterministic parity cases shared by the golden generator and the tests.

Each case is a dict with ``image`` (H, W, C) float64, ``labels`` (H, W)
uint8, ``guide`` ((H, W, 2) float64 or None), ``params`` (FillParams
keyword dict) and ``tracked`` (bool).  The first group restates the
reference's own engine/tracker test scenes (pkg/tests/test_engine.py,
test_tracker.py, test_acceptance.py); the second group is randomized stress
on the decision path (rotated balls at arbitrary guide angles, mu in
{0, finite, inf}, every order, periodic x, Bystander islands).
"""

from __future__ import annotations

import math

import numpy as np

READABLE, BYSTANDER, INPAINT = 0, 128, 255


def _block(H, W, j0, j1, i0, i1):
    lab = np.zeros((H, W), dtype=np.uint8)
    lab[j0:j1, i0:i1] = INPAINT
    return lab


def _case(name, image, labels, guide=None, tracked=True, **params):
    return dict(name=name, image=np.ascontiguousarray(image, dtype=np.float64),
                labels=np.ascontiguousarray(labels, dtype=np.uint8),
                guide=None if guide is None else np.ascontiguousarray(guide, dtype=np.float64),
                params=params, tracked=tracked)


def reference_scenes():
    """Scenes of the reference test-suite (file:line in each name)."""
    out = []
    lab = _block(20, 20, 5, 15, 5, 15)
    out.append(_case("onion_block test_engine.py:144", np.full((20, 20, 3), 0.25), lab,
                     tracked=False, order="onion"))
    lab = np.array([[READABLE, INPAINT, INPAINT, READABLE]], dtype=np.uint8)
    img = np.zeros((1, 4, 1))
    img[0, 3, 0] = 0.9
    out.append(_case("snapshot test_engine.py:156", img, lab, tracked=False, r=1, order="onion"))
    rng = np.random.default_rng(7)
    img = rng.random((24, 24, 3))
    lab = _block(24, 24, 8, 16, 8, 16)
    img[lab == INPAINT] = 0.0
    out.append(_case("rot_g0 test_engine.py:170", img, lab, tracked=False))
    out.append(_case("axis_g0 test_engine.py:170", img, lab, tracked=False, neighborhood="axis_ball"))
    rng = np.random.default_rng(3)
    img = rng.random((30, 30, 3))
    lab = _block(30, 30, 9, 21, 7, 23)
    img[lab == INPAINT] = 0.0
    g = np.zeros((30, 30, 2))
    g[:, :, 0] = 0.7
    out.append(_case("determinism test_engine.py:180", img, lab, g, tracked=False))
    rng = np.random.default_rng(11)
    img = rng.uniform(0.2, 0.6, size=(26, 26, 3))
    lab = _block(26, 26, 6, 20, 6, 20)
    img[lab == INPAINT] = 0.0
    out.append(_case("hull test_engine.py:192", img, lab, tracked=False, order="onion"))
    lab = np.zeros((12, 31), dtype=np.uint8)
    lab[6:, :] = INPAINT
    img = np.zeros((12, 31, 1))
    img[:6, :, 0] = 0.8
    out.append(_case("flat_front test_engine.py:226", img, lab, tracked=False, order="smart"))
    rng = np.random.default_rng(5)
    img = rng.random((20, 20, 1))
    lab = _block(20, 20, 6, 14, 6, 14)
    img[lab == INPAINT] = 0.0
    out.append(_case("dt_latch test_engine.py:234", img, lab, np.zeros((20, 20, 2)),
                     tracked=False, order="smart_with_data_term"))
    lab = _block(14, 40, 5, 9, 4, 36)
    img = np.full((14, 40, 1), 0.6)
    img[lab == INPAINT] = 0.0
    g = np.zeros((14, 40, 2))
    g[:, :20, 0] = 1.0
    out.append(_case("dt_defer test_engine.py:248", img, lab, g, tracked=False,
                     order="smart_with_data_term"))
    lab = np.full((7, 7), BYSTANDER, dtype=np.uint8)
    lab[:3, :3] = READABLE
    lab[3, 3] = INPAINT
    img = np.zeros((7, 7, 1))
    img[:3, :3, 0] = 0.45
    out.append(_case("deadlock_mean test_engine.py:263", img, lab, tracked=False, r=1, order="onion"))
    lab = np.zeros((8, 12), dtype=np.uint8)
    lab[4:, :] = INPAINT
    img = np.full((8, 12, 1), 0.3)
    img[lab == INPAINT] = 0.0
    th = math.radians(10.0)
    g = np.zeros((8, 12, 2))
    g[..., 0] = math.cos(th)
    g[..., 1] = math.sin(th)
    out.append(_case("deadlock_chain test_engine.py:277", img, lab, g, tracked=False, order="smart"))
    lab = np.zeros((11, 11), dtype=np.uint8)
    lab[3:8, 3:8] = BYSTANDER
    lab[4:7, 4:7] = INPAINT
    img = np.full((11, 11, 1), 0.7)
    img[3:8, 3:8] = 0.0
    out.append(_case("unfillable_pocket test_engine.py:294", img, lab, tracked=False, order="onion"))
    out.append(_case("unfillable_all test_engine.py:309", np.zeros((5, 5, 2)),
                     np.full((5, 5), INPAINT, dtype=np.uint8), tracked=False))
    for kind in ("axis_ball", "rotated_ball"):
        H, W, th = 80, 120, math.radians(73.0)
        image = np.full((H, W, 1), 1.0)
        jj, ii = np.mgrid[0:H, 0:W]
        d = -math.sin(th) * (ii - W / 2) + math.cos(th) * (jj - H / 2)
        lab = np.zeros((H, W), dtype=np.uint8)
        lab[H // 2:, :] = INPAINT
        image[(np.abs(d) <= 2.0) & (lab == READABLE), 0] = 0.0
        g = np.zeros((H, W, 2))
        g[..., 0] = math.cos(th)
        g[..., 1] = math.sin(th)
        out.append(_case(f"kink_{kind} test_engine.py:379", image, lab, g, tracked=False,
                         order="onion", neighborhood=kind, mu=50.0))
    rng = np.random.default_rng(19)
    img = rng.random((28, 34, 3))
    lab = np.zeros((28, 34), dtype=np.uint8)
    lab[7:21, 9:27] = INPAINT
    lab[12:15, 14:17] = BYSTANDER
    img[lab != READABLE] = 0.0
    g = np.zeros((28, 34, 2))
    g[..., 0] = 0.8
    g[..., 1] = 0.2
    out.append(_case("trk_untracked test_tracker.py:81", img, lab, g, tracked=False))
    out.append(_case("trk_tracked test_tracker.py:81", img, lab, g, tracked=True))
    lab = np.zeros((14, 14), dtype=np.uint8)
    lab[2:12, 2:12] = INPAINT
    img = np.full((14, 14, 1), 0.9)
    img[lab == INPAINT] = 0.0
    out.append(_case("trk_threads test_tracker.py:101", img, lab, tracked=True, order="onion"))
    lab = np.zeros((10, 12), dtype=np.uint8)
    lab[3:7, :3] = INPAINT
    lab[3:7, 9:] = INPAINT
    img = np.full((10, 12, 1), 0.2)
    img[lab == INPAINT] = 0.0
    out.append(_case("trk_periodic test_tracker.py:143", img, lab, tracked=True, order="onion",
                     periodic_x=True))
    return out


def islands_labels(rng, lo=24, hi=97):
    """Random elliptic holes with Bystander islands (cf. test_acceptance.py:175-199)."""
    H = int(rng.integers(lo, hi))
    W = int(rng.integers(lo, hi))
    lab = np.zeros((H, W), dtype=np.uint8)
    jj, ii = np.mgrid[0:H, 0:W]
    for _ in range(int(rng.integers(1, 4))):
        cy, cx = rng.uniform(0, H), rng.uniform(0, W)
        ry, rx = rng.uniform(3, H / 2), rng.uniform(3, W / 2)
        lab[((jj - cy) / ry) ** 2 + ((ii - cx) / rx) ** 2 <= 1.0] = INPAINT
    inp = np.argwhere(lab == INPAINT)
    for _ in range(int(rng.integers(1, 4))):
        if inp.size == 0:
            break
        j, i = inp[rng.integers(0, len(inp))]
        lab[j:j + int(rng.integers(1, 4)), i:i + int(rng.integers(1, 4))] = BYSTANDER
    for _ in range(int(rng.integers(0, 3))):
        lab[rng.integers(0, H), rng.integers(0, W)] = BYSTANDER
    return lab


def random_scenes(n=40, seed=1837, lo=16, hi=64):
    """Randomized decision-path stress: every order, ball, mu regime and g source."""
    rng = np.random.default_rng(seed)
    out = []
    orders = ("onion", "smart", "smart_with_data_term")
    for k in range(n):
        lab = islands_labels(rng, lo, hi)
        H, W = lab.shape
        C = int(rng.integers(1, 5))
        img = rng.uniform(size=(H, W, C))
        img[lab == INPAINT] = 0.0
        r = int(rng.integers(1, 7))
        mu = float(rng.choice([0.0, 10.0, 50.0, 100.0, math.inf]))
        order = orders[k % 3]
        nb = "axis_ball" if k % 4 == 3 else "rotated_ball"
        periodic = bool(k % 5 == 0)
        gmode = k % 4
        guide = None
        extra = {}
        if gmode == 0:
            extra = dict(g_source="fixed", g_fixed=(float(rng.uniform(-1, 1)), float(rng.uniform(-1, 1))))
        elif gmode == 1:
            extra = dict(g_source="fixed", g_fixed=(0.6, 0.8))
        elif gmode == 2:
            ang = rng.uniform(0, 2 * math.pi, size=(H, W))
            mag = rng.uniform(0, 1, size=(H, W)) * (rng.uniform(size=(H, W)) < 0.6)
            guide = np.stack([mag * np.cos(ang), mag * np.sin(ang)], axis=-1)
        out.append(_case(f"rand{k}", img, lab, guide, tracked=bool(k % 2 == 0), r=r, mu=mu,
                         order=order, neighborhood=nb, periodic_x=periodic, **extra))
    return out


def guide_cases(n=12, seed=303):
    """Random spline sets over random label maps for the rasteriser."""
    rng = np.random.default_rng(seed)
    out = []
    for k in range(n):
        lab = islands_labels(rng, 20, 90)
        H, W = lab.shape
        polys, dirs, kinds, raw = [], [], [], []
        for s in range(int(rng.integers(0, 5))):
            kind = "bezier" if rng.uniform() < 0.5 else "polyline"
            if kind == "bezier":
                pts = rng.uniform(-5, max(H, W) + 5, size=(3 * int(rng.integers(1, 3)) + 1, 2))
            else:
                pts = rng.uniform(-5, max(H, W) + 5, size=(int(rng.integers(2, 5)), 2))
                if k == 0 and s == 0:
                    pts = np.array([[3.0, 4.0], [3.0, 4.0 + 1e-9], [10.0, 12.0]])
            ang = rng.uniform(0, 2 * math.pi)
            mag = rng.uniform(0, 1)
            raw.append(dict(points=pts, kind=kind, direction=(mag * math.cos(ang), mag * math.sin(ang))))
        eta = float(rng.choice([3.0, 1.5, 4.0]))
        out.append(dict(name=f"gf{k}", labels=lab, splines=raw, eta=eta))
    return out


def edge_block():
    """test_guide.py _vertical_edge_block analogue: a vertical colour edge with an
    Inpaint block across it (coherence-direction fixtures)."""
    H, W = 64, 64
    img = np.zeros((H, W, 3))
    img[:, 30:, :] = 1.0
    img[:, :, 1] *= 0.5
    lab = _block(H, W, 20, 40, 22, 42)
    img[lab == INPAINT] = 0.0
    return img, lab


def coherence_scenes(n=10, seed=4242):
    """g_source = modified_structure_tensor (engine.py:243-249): the coherence-transport
    preset (engine.py:66-76: r=5, axis ball, onion) on an edge scene and random
    islands, plus smart-order / rotated-ball variants (order then reads g)."""
    rng = np.random.default_rng(seed)
    out = []
    img, lab = edge_block()
    ct = dict(r=5, neighborhood="axis_ball", order="onion", g_source="modified_structure_tensor")
    out.append(_case("ct_edge preset", img, lab, tracked=True, **ct))
    out.append(_case("ct_edge preset untracked", img, lab, tracked=False, **ct))
    out.append(_case("ct_edge smart rotated", img, lab, tracked=True, r=3, mu=50.0, order="smart",
                     neighborhood="rotated_ball", g_source="modified_structure_tensor"))
    for k in range(n):
        lab = islands_labels(rng, 20, 56)
        H, W = lab.shape
        C = int(rng.integers(1, 5))
        img = rng.uniform(size=(H, W, C))
        img[lab == INPAINT] = 0.0
        if k < n - 2:
            p = dict(ct, r=int(rng.choice([3, 4, 5])), mu=float(rng.choice([10.0, 50.0, 100.0, math.inf])),
                     sigma=float(rng.choice([1.0, 2.0])), rho=float(rng.choice([2.0, 4.0])))
        else:
            p = dict(r=3, mu=50.0, order="smart", neighborhood="rotated_ball",
                     g_source="modified_structure_tensor")
        out.append(_case(f"ct_rand{k}", img, lab, tracked=bool(k % 2 == 0), **p))
    # periodic x, data-term order, and a Bystander moat (unfillable fallback)
    lab = islands_labels(rng, 24, 48)
    H, W = lab.shape
    img = rng.uniform(size=(H, W, 3))
    img[lab == INPAINT] = 0.0
    out.append(_case("ct_periodic", img, lab, tracked=True, periodic_x=True, **ct))
    out.append(_case("ct_periodic untracked", img, lab, tracked=False, periodic_x=True, **ct))
    out.append(_case("ct_data_term", img, lab, tracked=True, r=3, mu=50.0,
                     order="smart_with_data_term", c2=0.5, neighborhood="rotated_ball",
                     g_source="modified_structure_tensor"))
    lab = np.zeros((40, 44), dtype=np.uint8)
    lab[6:30, 8:36] = INPAINT
    lab[14:22, 16:28] = BYSTANDER
    lab[17:19, 21:23] = INPAINT  # pocket cut off by the Bystander moat
    img = rng.uniform(size=(40, 44, 2))
    img[lab == INPAINT] = 0.0
    out.append(_case("ct_moat", img, lab, tracked=True, **ct))
    # smart / data-term order on the smooth edge scene: confidences far from
    # ties, so the order must be bit-exact (no near-tie excuse)
    img, lab = edge_block()
    out.append(_case("ct_edge data_term", img, lab, tracked=True, r=3, mu=50.0,
                     order="smart_with_data_term", c2=0.5, neighborhood="rotated_ball",
                     g_source="modified_structure_tensor"))
    out.append(_case("ct_edge smart untracked", img, lab, tracked=False, r=4, mu=100.0,
                     order="smart", neighborhood="rotated_ball",
                     g_source="modified_structure_tensor"))
    return out


def deadlock_scenes(size=256, thetas=(10.0, 25.0, 40.0, 73.0), mus=(50.0, 100.0), seed=2019):
    """SURVEY.md Appendix B / section 7 hard part 2: half-planes with a rotated
    guide, smart order -- the reference's deadlock-chain scene
    (test_engine.py:277-291) at 256x256.  Low angles fill one pixel per
    shell through the deadlock guard for 16-22K shells."""
    out = []
    H = W = size
    jj, ii = np.mgrid[0:H, 0:W].astype(np.float64)
    base = np.stack([0.5 + 0.3 * np.sin(ii / (9.0 + 4.0 * c) + jj / (13.0 + 3.0 * c) + seed % 7 + c)
                     for c in range(3)], axis=-1)  # smooth: the fixtures compress
    for th_deg in thetas:
        for mu in mus:
            lab = np.zeros((H, W), dtype=np.uint8)
            lab[H // 2:, :] = INPAINT
            img = base.copy()
            img[lab == INPAINT] = 0.0
            th = math.radians(th_deg)
            g = np.zeros((H, W, 2))
            g[..., 0] = math.cos(th)
            g[..., 1] = math.sin(th)
            out.append(_case(f"halfplane_{th_deg:g}deg_mu{mu:g}", img, lab, g, tracked=True,
                             r=3, mu=mu, order="smart", neighborhood="rotated_ball"))
    return out


def detect_scenes(seed=77):
    """Automatic-detection scenes: the reference test scenes (test_guide.py:16-36,
    200-209) plus random edge images around rectangular holes."""
    out = []
    jj, ii = np.mgrid[0:100, 0:100]
    img = np.where(jj >= ii, 1.0, 0.5)[..., None]
    lab = np.zeros((100, 100), dtype=np.uint8)
    lab[50:, :] = INPAINT
    img[lab != 0] = 0.0
    out.append(("half_plane_45", img, lab))
    lab = np.zeros((60, 60), dtype=np.uint8)
    lab[24:36, 24:36] = INPAINT
    img = np.zeros((60, 60, 3))
    img[:, 30:, :] = 1.0
    img[lab == INPAINT] = 0.0
    out.append(("vertical_edge_block", img, lab))
    img = np.where(jj >= 37.5, 1.0, 0.5)[..., None]
    lab = np.zeros((100, 100), dtype=np.uint8)
    lab[50:, :] = INPAINT
    img[lab != 0] = 0.0
    out.append(("parallel_edge", img, lab))
    rng = np.random.default_rng(seed)
    for k in range(4):
        H, W = int(rng.integers(70, 130)), int(rng.integers(70, 130))
        y, x = np.mgrid[0:H, 0:W].astype(np.float64)
        img = np.zeros((H, W, 3))
        for c in range(3):
            a = rng.uniform(0, np.pi)
            img[..., c] = np.where(np.cos(a) * (x - W / 2) + np.sin(a) * (y - H / 2) > rng.uniform(-5, 5),
                                   rng.uniform(0.6, 1.0), rng.uniform(0.0, 0.4))
        img += rng.uniform(0, 0.02, size=img.shape)
        lab = np.zeros((H, W), dtype=np.uint8)
        j0, i0 = int(H * 0.4), int(W * 0.4)
        lab[j0:j0 + int(rng.integers(8, 16)), i0:i0 + int(rng.integers(8, 16))] = INPAINT
        if k % 2:
            lab[j0 + 2:j0 + 4, i0 + 2:i0 + 4] = BYSTANDER
        img[lab == INPAINT] = 0.0
        out.append((f"random_edges_{k}", img, lab))
    return out
