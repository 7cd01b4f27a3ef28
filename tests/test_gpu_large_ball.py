"""Balls beyond the persistent kernels' tables (r > GF_MAX_RADIUS = 12).

The reference accepts any r >= 1 (engine.py:51-52).  Such fills take the
shell-by-shell device loop with the large-ball sampler (gf_sample_points:
tables and the numpy pairwise plan in HBM, any number of leaves).  Checked
against the oracle on the same inputs: fill order, frontier sets and report
rows bit-exact, values exact (the f64 colour path, numpy's einsum order).
"""

import math

import numpy as np
import pytest

from oracle import guidefill_oracle as orc
from paper_1611_05319_b200 import FillParams, engine

pytestmark = pytest.mark.gpu


def _scene(seed, H=44, W=52, C=3):
    rng = np.random.default_rng(seed)
    lab = np.zeros((H, W), dtype=np.uint8)
    lab[14:30, 10:42] = 255
    lab[20:23, 18:21] = 128
    img = rng.uniform(size=(H, W, C))
    img[lab == 255] = 0.0
    th = rng.uniform(0, math.pi)
    guide = np.zeros((H, W, 2))
    guide[lab == 255] = (0.9 * math.cos(th), 0.9 * math.sin(th))
    return img, lab, guide


CASES = [
    dict(r=13, mu=50.0, order="smart", neighborhood="rotated_ball"),
    dict(r=13, mu=math.inf, order="smart", neighborhood="rotated_ball"),
    dict(r=16, mu=100.0, order="onion", neighborhood="axis_ball"),
    dict(r=14, mu=50.0, order="smart_with_data_term", c2=0.3, neighborhood="rotated_ball"),
]


@pytest.mark.parametrize("k", range(len(CASES)))
@pytest.mark.parametrize("tracked", [True, False])
def test_large_ball_matches_oracle(k, tracked):
    img, lab, guide = _scene(100 + k, C=1 + k % 3)
    p = FillParams(**CASES[k])
    u, rep, maps = engine._run_fill(img, lab, guide, p, tracked=tracked, order_log=True)
    ref = orc.fill(img, lab, guide, orc.Params.of(p), tracked=tracked)
    assert np.array_equal(maps["fillshell"], ref["fillshell"].reshape(lab.shape))
    assert np.array_equal(maps["enter"], ref["enter"].reshape(lab.shape))
    assert [tuple(r) for r in rep.rows] == [tuple(r) for r in ref["rows"]]
    assert rep.deadlock_fills == ref["deadlock_fills"]
    assert np.array_equal(u, ref["u"]), float(np.abs(u - ref["u"]).max())


def test_large_ball_single_pixel_api():
    """engine.confidence / fill_color (engine.py:202-221) at r = 15."""
    img, lab, guide = _scene(7)
    p = FillParams(r=15, mu=60.0)
    pt, g = (20, 16), (0.6, 0.5)
    got = engine.confidence(pt, img, lab, g, p)
    vals, rw, tw = orc.point_sample(img, lab, pt, np.array(g), orc.Params.of(p))
    assert got == float(rw[0] / tw[0])
    col, ok = engine.fill_color(pt, img, lab, g, p)
    assert ok and np.array_equal(np.asarray(col), vals[0])


def test_large_ball_coherence_transport():
    """g from the masked structure tensor with r = 13: gf_coherence_fill declines
    the ball (its tables stop at r = 12) and the shell loop takes over."""
    img, lab, _ = _scene(11)
    p = FillParams.coherence_transport(r=13)
    u, rep, maps = engine._run_fill(img, lab, None, p, tracked=True, order_log=True)
    ref = orc.fill(img, lab, None, orc.Params.of(p), tracked=True)
    assert np.array_equal(maps["fillshell"], ref["fillshell"].reshape(lab.shape))
    assert [tuple(r) for r in rep.rows] == [tuple(r) for r in ref["rows"]]
    assert np.array_equal(u, ref["u"])
