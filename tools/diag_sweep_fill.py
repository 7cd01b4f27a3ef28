"""First differing pixel of a sweep_fill scene: the oracle's sample at it."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases  # noqa: E402
from oracle import guidefill_oracle as orc  # noqa: E402
from paper_1611_05319_b200 import FillParams, engine  # noqa: E402

target, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
for it in range(target + 1):
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
fs = maps["fillshell"]
diff = np.abs(u - ref["u"]).max(axis=2) > 1e-4
jj, ii = np.nonzero(diff)
k = fs[jj, ii].min()
sel = fs[jj, ii] == k
print(p, tracked, "first differing shell", k, "pixels", list(zip(ii[sel].tolist(), jj[sel].tolist()))[:5])
state = img.copy()
fsr = ref["fillshell"].reshape(H, W)
earlier = (fsr >= 0) & (fsr < k)
state[earlier] = ref["u"][earlier]
readable = (lab == 0) | earlier
offs = orc.disk_offsets(p.r)[1:]
for i, j in list(zip(ii[sel].tolist(), jj[sel].tolist()))[:3]:
    g = guide[j, i] if guide is not None else np.array(p.g_fixed)
    vals, rw, tw = orc.sample_frontier(state, readable, np.array([float(i)]), np.array([float(j)]),
                                       g[None, :], orc.Params.of(p), offs)
    print("px", (i, j), "g", g.tolist(), "rw", rw[0], "tw", tw[0], "oracle vals", vals[0].tolist(),
          "final oracle", ref["u"][j, i].tolist(), "gpu", u[j, i].tolist(),
          "readable nbrs", int(sum(readable[j + dj, i + di] for di in (-1, 0, 1) for dj in (-1, 0, 1)
                                    if 0 <= j + dj < H and 0 <= i + di < W)))
