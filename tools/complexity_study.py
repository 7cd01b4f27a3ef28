"""The paper's complexity figure (T(N), P(N), Section 6) on one B200.

Stripe family omega = [0,4]x[0,1], D = [0.4,3.96]x[0.2,0.8], rendered on the
device; tracked up to N = 1e8 px, untracked up to 1.6e7 px (every untracked
shell rescans the whole lattice).  Fits T ~ N^alpha and P ~ N^beta over the
paper's range (N <= 1e6) and over the whole sweep.
Usage: python tools/complexity_study.py [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_05319_b200 import harness  # noqa: E402

H_T = (50, 70, 100, 140, 200, 280, 400, 500, 1000, 2000, 3000, 5000)
H_U = (50, 70, 100, 140, 200, 280, 400, 500, 1000, 2000)


def fits(rows, nmax=None):
    pts = [r for r in rows if nmax is None or r["N"] <= nmax]
    return {"alpha_time": harness.fit_power_law([(r["N"], r["seconds"]) for r in pts]).alpha,
            "beta_threads": harness.fit_power_law([(r["N"], r["threads_max"]) for r in pts]).alpha,
            "n_points": len(pts), "N_max": max(r["N"] for r in pts)}


def main():
    out = {"tracked": harness.scaling_study(harness.stripe_family(H_T), tracked=True),
           "untracked": harness.scaling_study(harness.stripe_family(H_U), tracked=False)}
    out["fits"] = {f"{k}_paper_range": fits(out[k], 1_000_000) for k in ("tracked", "untracked")}
    out["fits"].update({f"{k}_full": fits(out[k]) for k in ("tracked", "untracked")})
    out["paper"] = {"tracked": {"alpha": 0.54, "beta": 0.5}, "untracked": {"alpha": 1.10, "beta": 1.0},
                    "range": "N ~ 1e4 .. 1e6, GeForce GTX 970M (PAPER.md:659, :816)"}
    for k in ("tracked", "untracked"):
        for r in out[k]:
            print(k, r["N"], "D", r["inpaint_px"], "shells", r["iterations"], "threads_max",
                  r["threads_max"], "ms %.3f" % (r["seconds"] * 1e3), flush=True)
    print(json.dumps(out["fits"], indent=1))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
