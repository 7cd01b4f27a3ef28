"""Golden fixtures for the continuum-limit module, made by running the
REFERENCE (pkg/src/guidefill/limits.py) in the build container:

    python tests/golden/make_limits_golden.py

Writes tests/golden/limits_golden.npz: half balls, limit directions, an
angle curve, integral limits, and two small convergence studies.
"""

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import refimport  # noqa: E402

DIRS = [("axis_ball", 3, 1.0, (0.0, 1.0)), ("rotated_ball", 3, 1.0, (0.3, 0.8)),
        ("rotated_ball", 5, 50.0, (-0.6, 0.2)), ("axis_ball", 4, math.inf, (0.9, 0.1)),
        ("rotated_ball", 3, math.inf, (0.5, 0.5)), ("rotated_ball", 2, 10.0, (0.05, 1.0))]
INTEG = [(1.0, (0.3, 0.8)), (5.0, (0.0, 1.0)), (math.inf, (-0.4, 0.7)), (20.0, (0.9, 0.2))]
RES = (16, 32, 64)


def smooth(x):
    return np.sin(2.0 * np.pi * np.asarray(x))


def step(x):
    return np.where(np.mod(np.asarray(x), 1.0) < 0.5, 0.0, 1.0)


def main():
    refimport.load()
    from guidefill import limits

    out = {}
    for k, (kind, r, mu, g) in enumerate(DIRS):
        hb = limits.half_ball(kind, r, g)
        pred = limits.limit_direction(kind, r, mu, g)
        out[f"hb{k}"] = hb.points
        out[f"ld{k}"] = np.array([pred.g_star[0], pred.g_star[1], pred.theta_star])
    th, ts = limits.limit_angle_curve("rotated_ball", 3, 1.0, samples=9)
    out["curve"] = np.stack([th, ts])
    for k, (mu, g) in enumerate(INTEG):
        pred = limits.integral_limit_direction(mu, g)
        out[f"il{k}"] = np.array([pred.g_star[0], pred.g_star[1], pred.theta_star])
    for name, trace, kind, g in (("smooth", smooth, "rotated_ball", (0.0, 1.0)),
                                 ("step", step, "rotated_ball", (0.4, 0.9)),
                                 ("axis", smooth, "axis_ball", (0.3, 0.95))):
        st = limits.convergence_study(trace, kind=kind, r=3, mu=1.0, g=g, resolutions=RES)
        out[f"cs_{name}"] = np.array([[st["errors"][n][p] for p in (1, 2, math.inf)] for n in RES])
        out[f"cs_{name}_theta"] = np.float64(st["theta_star_rad"])
        print(name, out[f"cs_{name}"].tolist())
    np.savez_compressed(os.path.join(HERE, "limits_golden.npz"), **out)


if __name__ == "__main__":
    main()
