"""Complexity-study harness vs the reference harness.

Golden fixtures: tests/golden/harness_golden.npz, made by running the
reference's own harness (tests/golden/make_harness_golden.py).  CPU tests pin
the rasteriser and the fit; GPU tests pin the device rasteriser and the
scaling-study rows of the B200 engine, and reproduce the exponent test of
the reference's acceptance suite (test_acceptance.py:230-244)."""

import math
import os

import numpy as np
import pytest

from paper_1611_05319_b200 import harness

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "harness_golden.npz"))
SPECS = [
    dict(),
    dict(geometry="step", theta_deg=30.0, resolution=(64, 48)),
    dict(theta_deg=0.0, colors=((0.1, 0.2, 0.9), (0.8, 0.7, 0.05)), resolution=(90, 33)),
    dict(omega=(0.0, 4.0, 0.0, 1.0), domain=(0.4, 3.96, 0.2, 0.8), theta_deg=0.0,
         resolution=(120, 30)),
    dict(theta_deg=135.0, half_width=0.11, resolution=(57, 71)),
]
HEIGHTS = (12, 16, 20, 26)


@pytest.mark.parametrize("k", range(len(SPECS)))
def test_render_problem_matches_reference(k):
    image, labels, truth = harness.render_problem(harness.SyntheticProblem(**SPECS[k]))
    assert image.tobytes() == GOLD[f"r{k}_image"].tobytes()
    assert image.shape == GOLD[f"r{k}_image"].shape
    assert np.array_equal(labels, GOLD[f"r{k}_labels"]) and labels.dtype == np.uint8
    assert truth.tobytes() == GOLD[f"r{k}_truth"].tobytes()
    assert harness.shell_count(harness.SyntheticProblem(**SPECS[k])) == int(GOLD[f"r{k}_shells"])


def test_fit_power_law_matches_reference():
    fit = harness.fit_power_law([(1e4, 0.02), (3e4, 0.031), (1e5, 0.06), (4e5, 0.13)])
    assert np.array_equal(np.array([fit.amplitude, fit.alpha, fit.residual]), GOLD["fit"])
    with pytest.raises(harness.DegenerateFitError):
        harness.fit_power_law([(10, 1.0), (10, 2.0)])
    with pytest.raises(ValueError):
        harness.fit_power_law([(10, 1.0)])
    with pytest.raises(ValueError):
        harness.fit_power_law([(10, 1.0), (0, 2.0)])


@pytest.mark.parametrize("kw,msg", [
    (dict(omega=(1.0, 0.0, 0.0, 1.0)), "omega rectangle is empty"),
    (dict(domain=(-1.0, 0.8, -0.3, 0.3)), "strictly inside"),
    (dict(geometry="blob"), "unknown geometry"),
    (dict(half_width=0.0), "half_width must be positive"),
    (dict(resolution=(1, 10)), "at least 2x2"),
    (dict(colors=(0.0, 1.0, 0.5)), "exactly two tones"),
    (dict(colors=((0.0, 1.0), 0.5)), "same channel count"),
])
def test_spec_errors(kw, msg):
    with pytest.raises(harness.SpecError, match=msg):
        harness.render_problem(harness.SyntheticProblem(**kw))


def test_stripe_family_shapes():
    fam = harness.stripe_family((50, 500))
    assert [p.resolution for p in fam] == [(200, 50), (2000, 500)]
    assert harness.scaling_csv([{"N": 10, "seconds": 0.5, "threads_max": 3, "iterations": 2}]) \
        == "N,seconds,threads_max,iterations\n10,0.5,3,2\n"


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(SPECS)))
def test_render_problem_device_is_bit_identical(k):
    import torch

    spec = harness.SyntheticProblem(**SPECS[k])
    img, lab = harness.render_problem_device(spec)
    assert img.dtype == torch.float64 and img.is_cuda
    assert img.cpu().numpy().tobytes() == GOLD[f"r{k}_image"].tobytes()
    assert np.array_equal(lab.cpu().numpy(), GOLD[f"r{k}_labels"])


@pytest.mark.gpu
@pytest.mark.parametrize("tracked", [True, False])
def test_scaling_study_rows_match_reference(tracked):
    rows = harness.scaling_study(harness.stripe_family(HEIGHTS), tracked=tracked, repeats=1)
    got = np.array([[r["N"], r["threads_max"], r["iterations"],
                     -1 if r["work_total"] is None else r["work_total"]] for r in rows])
    assert np.array_equal(got, GOLD["study_t" if tracked else "study_u"])
    assert all(r["seconds"] > 0 for r in rows)


@pytest.mark.gpu
def test_complexity_exponents_on_gpu():
    """test_acceptance.py:230-244 on the B200 engine: lane-demand exponents
    beta ~ 0.5 tracked, ~ 1.0 untracked over N in [1e4, 1e6]."""
    fam = harness.stripe_family()
    rows_t = harness.scaling_study(fam, tracked=True, repeats=1)
    rows_u = harness.scaling_study(fam, tracked=False, repeats=1)
    beta_t = harness.fit_power_law([(r["N"], r["threads_max"]) for r in rows_t]).alpha
    beta_u = harness.fit_power_law([(r["N"], r["threads_max"]) for r in rows_u]).alpha
    assert 0.4 <= beta_t <= 0.6
    assert 0.95 <= beta_u <= 1.05
    assert all(math.isfinite(r["seconds"]) for r in rows_t + rows_u)
