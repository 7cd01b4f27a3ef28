"""Random sweep of balls with r > 12 (large-ball sampler + shell loop) against the oracle."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases  # noqa: E402
from oracle import guidefill_oracle as orc  # noqa: E402
from paper_1611_05319_b200 import FillParams, engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
bad = 0
for it in range(n):
    lab = cases.islands_labels(rng, 30, 70)
    H, W = lab.shape
    C = int(rng.integers(1, 5))
    img = rng.uniform(size=(H, W, C))
    img[lab == 255] = 0.0
    th = rng.uniform(0, math.pi, size=(H, W))
    guide = np.stack([np.cos(th), np.sin(th)], -1) * rng.choice([0.0, 0.5, 1.0], size=(H, W))[..., None]
    guide[lab != 255] = 0.0
    src = ["guide_field", "fixed", "modified_structure_tensor"][it % 3]
    p = FillParams(r=int(rng.integers(13, 21)), mu=float(rng.choice([0.0, 30.0, 100.0, math.inf])),
                   order=["onion", "smart", "smart_with_data_term"][int(rng.integers(0, 3))],
                   c2=float(rng.uniform(0.1, 0.9)),
                   neighborhood=["rotated_ball", "axis_ball"][int(rng.integers(0, 2))],
                   g_source=src, g_fixed=(0.6, 0.8), periodic_x=bool(it % 4 == 1))
    tracked = bool(it % 3 != 2)
    gv = guide if src == "guide_field" else None
    u, rep, maps = engine._run_fill(img, lab, gv, p, tracked=tracked, order_log=True)
    ref = orc.fill(img, lab, gv, orc.Params.of(p), tracked=tracked)
    ok = (np.array_equal(maps["fillshell"], ref["fillshell"].reshape(H, W)) and
          [tuple(r) for r in rep.rows] == [tuple(r) for r in ref["rows"]] and
          np.array_equal(u, ref["u"]))
    if not ok:
        bad += 1
        print(f"it {it}: MISMATCH {p} tracked={tracked} C={C} {H}x{W} max|du|={np.abs(u - ref['u']).max():.2e}",
              flush=True)
print(f"{n - bad}/{n} ok")
