"""Golden fixtures for the complexity-study harness, made by running the
REFERENCE harness (pkg/src/guidefill/harness.py) in the build container:

    python tests/golden/make_harness_golden.py

Writes tests/golden/harness_golden.npz: rendered problems (image, labels),
shell counts, a power-law fit, and scaling_study rows (N, threads_max,
iterations, work_total) of a small stripe family, tracked and untracked.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import refimport  # noqa: E402

SPECS = [
    dict(),  # the dataclass defaults: 73 degree line, 200x100
    dict(geometry="step", theta_deg=30.0, resolution=(64, 48)),
    dict(theta_deg=0.0, colors=((0.1, 0.2, 0.9), (0.8, 0.7, 0.05)), resolution=(90, 33)),
    dict(omega=(0.0, 4.0, 0.0, 1.0), domain=(0.4, 3.96, 0.2, 0.8), theta_deg=0.0,
         resolution=(120, 30)),
    dict(theta_deg=135.0, half_width=0.11, resolution=(57, 71)),
]
HEIGHTS = (12, 16, 20, 26)


def main():
    refimport.load()
    from guidefill import harness

    out = {}
    for k, kw in enumerate(SPECS):
        spec = harness.SyntheticProblem(**kw)
        image, labels, truth = harness.render_problem(spec)
        out[f"r{k}_image"] = image
        out[f"r{k}_labels"] = labels
        out[f"r{k}_truth"] = truth
        out[f"r{k}_shells"] = np.int64(harness.shell_count(spec))
    pts = [(1e4, 0.02), (3e4, 0.031), (1e5, 0.06), (4e5, 0.13)]
    fit = harness.fit_power_law(pts)
    out["fit"] = np.array([fit.amplitude, fit.alpha, fit.residual])
    fam = harness.stripe_family(HEIGHTS)
    for tracked in (True, False):
        rows = harness.scaling_study(fam, tracked=tracked)
        key = "study_t" if tracked else "study_u"
        out[key] = np.array([[r["N"], r["threads_max"], r["iterations"],
                              -1 if r["work_total"] is None else r["work_total"]] for r in rows],
                            dtype=np.int64)
        print(key, out[key].tolist())
    np.savez_compressed(os.path.join(HERE, "harness_golden.npz"), **out)


if __name__ == "__main__":
    main()
