"""Continuum-limit module vs the reference's limits.py.

Golden fixtures (tests/golden/limits_golden.npz) come from running the
reference itself (tests/golden/make_limits_golden.py).  The predictions are
host computations and must match bit for bit; the convergence studies fill
on the GPU, whose values agree with the reference within the fill tolerance,
and reproduce the reference acceptance test's orders
(test_acceptance.py:97-123)."""

import math
import os

import numpy as np
import pytest

from paper_1611_05319_b200 import limits

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "limits_golden.npz"))
DIRS = [("axis_ball", 3, 1.0, (0.0, 1.0)), ("rotated_ball", 3, 1.0, (0.3, 0.8)),
        ("rotated_ball", 5, 50.0, (-0.6, 0.2)), ("axis_ball", 4, math.inf, (0.9, 0.1)),
        ("rotated_ball", 3, math.inf, (0.5, 0.5)), ("rotated_ball", 2, 10.0, (0.05, 1.0))]
INTEG = [(1.0, (0.3, 0.8)), (5.0, (0.0, 1.0)), (math.inf, (-0.4, 0.7)), (20.0, (0.9, 0.2))]
RES = (16, 32, 64)


def smooth(x):
    return np.sin(2.0 * np.pi * np.asarray(x))


def step(x):
    return np.where(np.mod(np.asarray(x), 1.0) < 0.5, 0.0, 1.0)


@pytest.mark.parametrize("k", range(len(DIRS)))
def test_half_ball_and_limit_direction(k):
    kind, r, mu, g = DIRS[k]
    assert np.array_equal(limits.half_ball(kind, r, g).points, GOLD[f"hb{k}"])
    pred = limits.limit_direction(kind, r, mu, g)
    assert np.array_equal(np.array([*pred.g_star, pred.theta_star]), GOLD[f"ld{k}"])


def test_angle_curve_and_integral_limit():
    th, ts = limits.limit_angle_curve("rotated_ball", 3, 1.0, samples=9)
    assert np.array_equal(np.stack([th, ts]), GOLD["curve"])
    for k, (mu, g) in enumerate(INTEG):
        pred = limits.integral_limit_direction(mu, g)
        assert np.array_equal(np.array([*pred.g_star, pred.theta_star]), GOLD[f"il{k}"])
    assert limits.curve_to_csv([1.0], [2.5]) == "theta_deg,theta_star_deg\n1,2.5\n"


def test_limit_errors():
    with pytest.raises(ValueError, match="kind must be one of"):
        limits.half_ball("square", 3)
    with pytest.raises(ValueError, match="r must be >= 1"):
        limits.half_ball("axis_ball", 0)
    with pytest.raises(ValueError, match="nonzero guide direction"):
        limits.limit_direction("rotated_ball", 3, 1.0, (0.0, 0.0))
    with pytest.raises(ValueError, match="point into the unknown half"):
        limits.limit_direction("rotated_ball", 3, 1.0, (0.0, -1.0))
    with pytest.raises(ValueError, match="theta_star must lie"):
        limits.transport_solution(smooth, 0.0, [0.0], [0.0])
    with pytest.raises(limits.EmptySetError):
        limits.half_ball("rotated_ball", 1, (1.0, 0.05))
    assert limits.discrete_lp_error(np.array([3.0, -4.0]), 0.5, 2) == pytest.approx(2.5)
    assert limits.discrete_lp_error(np.array([3.0, -4.0]), 0.5, math.inf) == 4.0


@pytest.mark.gpu
@pytest.mark.parametrize("name,trace,kind,g", [("smooth", smooth, "rotated_ball", (0.0, 1.0)),
                                               ("step", step, "rotated_ball", (0.4, 0.9)),
                                               ("axis", smooth, "axis_ball", (0.3, 0.95))])
def test_convergence_study_matches_reference(name, trace, kind, g):
    st = limits.convergence_study(trace, kind=kind, r=3, mu=1.0, g=g, resolutions=RES)
    assert st["theta_star_rad"] == float(GOLD[f"cs_{name}_theta"])
    got = np.array([[st["errors"][n][p] for p in (1, 2, math.inf)] for n in RES])
    # the fill agrees with the reference within 1e-4 per pixel (fp32 colours):
    # every discrete norm of the difference moves by less than that
    assert float(np.abs(got - GOLD[f"cs_{name}"]).max()) <= 1e-4
    assert "N,p,error,order" in limits.study_to_csv(st)


@pytest.mark.gpu
def test_convergence_orders_on_gpu():
    """test_acceptance.py:97-123 on the B200 engine."""
    res = (128, 256, 512, 1024)
    sm = limits.convergence_study(smooth, kind="rotated_ball", r=3, mu=1.0, g=(0.0, 1.0),
                                  resolutions=res)
    assert all(0.8 <= o <= 1.2 for o in sm["orders"][math.inf])
    st = limits.convergence_study(step, kind="rotated_ball", r=3, mu=1.0, g=(0.0, 1.0),
                                  resolutions=res)
    assert all(o >= 0.3 for o in st["orders"][1])
    linf = [st["errors"][n][math.inf] for n in res]
    assert all(b / a >= 0.9 for a, b in zip(linf, linf[1:]))
