"""Randomised sweep of the persistent fill against the oracle (beyond the fixed
parity set): random islands, channels, guide fields with zero / partial /
unit magnitudes, fixed g, every order and ball, mu from 0 to inf, r up to 12,
periodic x, tracked and untracked.  Fill order, frontier sets and report rows
bit-exact, values within 1e-4.  (tools/sweep_fill.py runs the same sweep at
any size; 320 scenes passed on B200.)"""

import math

import numpy as np
import pytest

import cases
from oracle import guidefill_oracle as orc
from paper_1611_05319_b200 import FillParams, engine

pytestmark = pytest.mark.gpu


def _scene(rng, it):
    lab = cases.islands_labels(rng, 20, 72)
    H, W = lab.shape
    C = int(rng.integers(1, 5))
    img = rng.uniform(size=(H, W, C))
    img[lab == 255] = 0.0
    src = ["guide_field", "fixed", "guide_field"][it % 3]
    guide, kw = None, {}
    if src == "guide_field":
        th = rng.uniform(0, math.pi, size=(H, W))
        mag = rng.choice([0.0, 0.3, 0.97, 1.0], size=(H, W))
        guide = np.stack([np.cos(th) * mag, np.sin(th) * mag], axis=-1)
        guide[lab != 255] = 0.0
    else:
        t = rng.uniform(0, math.pi)
        kw["g_fixed"] = (math.cos(t), math.sin(t))
    p = FillParams(r=int(rng.integers(1, 13)), mu=float(rng.choice([0.0, 5.0, 50.0, 100.0, math.inf])),
                   order=["onion", "smart", "smart_with_data_term"][int(rng.integers(0, 3))],
                   c=float(rng.choice([0.05, 0.2])), c2=float(rng.uniform(0.1, 0.9)),
                   neighborhood=["rotated_ball", "axis_ball"][int(rng.integers(0, 2))],
                   g_source=src, periodic_x=bool(rng.integers(0, 4) == 0), **kw)
    return img, lab, guide, p, bool(rng.integers(0, 3) != 0)


def _check(img, lab, guide, p, tracked):
    u, rep, maps = engine._run_fill(img, lab, guide, p, tracked=tracked, order_log=True)
    ref = orc.fill(img, lab, guide, orc.Params.of(p), tracked=tracked)
    H, W = lab.shape
    assert np.array_equal(maps["fillshell"], ref["fillshell"].reshape(H, W)), p
    assert np.array_equal(maps["enter"], ref["enter"].reshape(H, W)), p
    assert [tuple(r) for r in rep.rows] == [tuple(r) for r in ref["rows"]], p
    assert float(np.abs(u - ref["u"]).max()) <= 1e-4, p


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_random_sweep():
    rng = np.random.default_rng(4242)
    for it in range(24):
        _check(*_scene(rng, it))


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_denormal_weights():
    """r = 1, mu = 100, a guided axis ball: coef = -5000, so most Eq. 3.2 weights
    are exactly 0 and the rest are denormals (rw = 5e-324): numpy's products
    round to multiples of 2^-1074 and the fill runs through the guard."""
    rng = np.random.default_rng(38)
    lab = np.zeros((40, 56), dtype=np.uint8)
    lab[12:28, 10:46] = 255
    img = rng.uniform(size=(40, 56, 1))
    img[lab == 255] = 0.0
    th = rng.uniform(0, math.pi, size=(40, 56))
    guide = np.stack([np.cos(th), np.sin(th)], axis=-1) * 0.97
    guide[lab != 255] = 0.0
    for order in ("smart", "smart_with_data_term"):
        p = FillParams(r=1, mu=100.0, order=order, c=0.2, c2=0.3, neighborhood="axis_ball")
        for tracked in (True, False):
            _check(img, lab, guide, p, tracked)
