"""Random sweep of the persistent fill (gf_fill) against the oracle: fill order,
frontier sets and rows bit-exact, values within 1e-4."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases  # noqa: E402
from oracle import guidefill_oracle as orc  # noqa: E402
from paper_1611_05319_b200 import FillParams, engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 99
rng = np.random.default_rng(seed)
bad = 0
for it in range(n):
    lab = cases.islands_labels(rng, 20, 80)
    H, W = lab.shape
    C = int(rng.integers(1, 5))
    img = rng.uniform(size=(H, W, C))
    img[lab == 255] = 0.0
    src = ["guide_field", "fixed", "guide_field"][it % 3]
    guide = None
    kw = {}
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
    tracked = bool(rng.integers(0, 3) != 0)
    u, rep, maps = engine._run_fill(img, lab, guide, p, tracked=tracked, order_log=True)
    ref = orc.fill(img, lab, guide, orc.Params.of(p), tracked=tracked)
    ok = (np.array_equal(maps["fillshell"], ref["fillshell"].reshape(H, W)) and
          np.array_equal(maps["enter"], ref["enter"].reshape(H, W)) and
          [tuple(r) for r in rep.rows] == [tuple(r) for r in ref["rows"]])
    err = float(np.abs(u - ref["u"]).max())
    if not ok or err > 1e-4:
        bad += 1
        print(f"it {it}: MISMATCH order_ok={ok} err={err:.2e} {p} tracked={tracked} C={C} {H}x{W}",
              flush=True)
        for j, i in np.argwhere(np.abs(u - ref["u"]).max(axis=2) > 1e-4)[:5]:
            print("   px", (int(i), int(j)), "gpu", u[j, i].tolist(), "oracle", ref["u"][j, i].tolist(),
                  "shell", int(maps["fillshell"][j, i]), "rep deadlocks", rep.deadlock_fills,
                  ref["deadlock_fills"], "unfillable", rep.unfillable, ref["unfillable"])
print(f"{n - bad}/{n} ok")
