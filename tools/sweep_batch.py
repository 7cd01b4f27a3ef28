"""Random sweep of the batched fill (several frames in one cooperative launch)
against one launch per frame: outputs, stats and report rows identical."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases  # noqa: E402
from paper_1611_05319_b200 import FillParams  # noqa: E402
from paper_1611_05319_b200._device import fill_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
bad = 0
for it in range(n):
    H, W = int(rng.integers(24, 80)), int(rng.integers(24, 80))
    N = int(rng.integers(2, 7))
    C = int(rng.integers(1, 5))
    labs = []
    for f in range(N):
        while True:
            lab = cases.islands_labels(rng, 10, 200)
            if lab.shape[0] >= H and lab.shape[1] >= W:
                break
        labs.append(lab[:H, :W].copy())
    if it % 4 == 0:
        labs[-1][:] = 0  # a frame with nothing to fill
    imgs = rng.uniform(size=(N, H, W, C)).astype(np.float32)
    t = rng.uniform(0, math.pi)
    p = FillParams(r=int(rng.integers(1, 8)), mu=float(rng.choice([0.0, 50.0, math.inf])),
                   order=["onion", "smart", "smart_with_data_term"][it % 3],
                   neighborhood=["rotated_ball", "axis_ball"][int(rng.integers(0, 2))],
                   g_source=["guide_field", "fixed"][it % 2], g_fixed=(math.cos(t), math.sin(t)),
                   periodic_x=bool(it % 5 == 1))
    guide = None
    if p.g_source == "guide_field":
        th = rng.uniform(0, math.pi, size=(N, H, W))
        guide = torch.from_numpy(np.stack([np.cos(th), np.sin(th)], -1) * 0.9).cuda()
    tracked = bool(it % 3 != 2)
    d_img = torch.from_numpy(imgs).cuda()
    d_lab = torch.from_numpy(np.stack(labs)).cuda()
    res = fill_device(d_img, d_lab, guide, p, tracked=tracked, rows_cap=H * W + 1)
    torch.cuda.synchronize()
    ok = True
    for f in range(N):
        one = fill_device(d_img[f:f + 1].contiguous(), d_lab[f:f + 1].contiguous(),
                          guide[f:f + 1].contiguous() if guide is not None else None, p,
                          tracked=tracked, rows_cap=H * W + 1)
        torch.cuda.synchronize()
        it_n = int(one["stats"][0][0])
        parts = dict(out=torch.equal(res["out"][f], one["out"][0]),
                     stats=torch.equal(res["stats"][f], one["stats"][0]),
                     rows=torch.equal(res["rows"][f, :it_n], one["rows"][0, :it_n]))
        if not all(parts.values()):
            ok = False
            print(f"it {it} frame {f}/{N}: batch != single {parts} ({p}, tracked={tracked}, C={C}, {H}x{W})")
            if not parts["out"]:
                d = (res["out"][f] != one["out"][0]).any(-1).nonzero()
                j, i = d[0].tolist()
                print("   first out diff", (i, j), res["out"][f][j, i].tolist(), one["out"][0][j, i].tolist(),
                      "label", int(d_lab[f, j, i]), "n diff", len(d))
    bad += not ok
print(f"{n - bad}/{n} ok")
