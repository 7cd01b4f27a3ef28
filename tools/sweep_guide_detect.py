"""Random sweeps: the guide-field raster (gf_guide_field) and spline detection
(gf_detect_edges + gf_structure_eigen + gf_trace_rays + host clustering)
against the oracles."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases  # noqa: E402
from oracle import detect_oracle as dor  # noqa: E402
from oracle import guidefill_oracle as orc  # noqa: E402
from paper_1611_05319_b200 import Spline, build_guide_field, guide  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 17)
bad = 0
for it in range(n):
    lab = cases.islands_labels(rng, 24, 120)
    H, W = lab.shape
    spl, polys, dirs = [], [], []
    for s in range(int(rng.integers(1, 6))):
        kind = ["polyline", "bezier"][int(rng.integers(0, 2))]
        npt = 4 if kind == "bezier" else int(rng.integers(2, 6))
        if kind == "bezier" and rng.integers(0, 2):
            npt = 7
        pts = np.column_stack([rng.uniform(-5, W + 5, npt), rng.uniform(-5, H + 5, npt)])
        th = rng.uniform(0, 2 * math.pi)
        d = (float(0.98 * math.cos(th)), float(0.98 * math.sin(th)))
        spl.append(Spline(id=f"s{s}", source="user", direction=d, points=pts.tolist(), kind=kind))
        polys.append(orc.polyline(pts, kind))
        dirs.append(d)
    eta = float(rng.choice([1.0, 3.0, 5.5]))
    got = build_guide_field(spl, lab, eta)
    ref = orc.guide_field(polys, dirs, lab, eta)
    if not np.array_equal(got, ref):
        bad += 1
        print(f"guide it {it}: {int((got != ref).any(-1).sum())} px differ", flush=True)
print(f"guide field: {n - bad}/{n} ok")
bad = 0
total = 0
for it in range(n):
    H, W = int(rng.integers(60, 140)), int(rng.integers(60, 140))
    jj, ii = np.mgrid[0:H, 0:W]
    img = np.zeros((H, W, 3))
    for _ in range(int(rng.integers(1, 4))):
        th = rng.uniform(0, math.pi)
        off = rng.uniform(-30, 30)
        side = (ii - W / 2) * math.cos(th) + (jj - H / 2) * math.sin(th) > off
        img[side] += rng.uniform(0.2, 0.5, size=3)
    img = np.clip(img + rng.normal(0, 0.01, img.shape), 0, 1)
    lab = np.zeros((H, W), dtype=np.uint8)
    cy, cx = H // 2 + int(rng.integers(-5, 6)), W // 2 + int(rng.integers(-5, 6))
    ry, rx = int(rng.integers(6, H // 4)), int(rng.integers(6, W // 4))
    lab[max(0, cy - ry):cy + ry, max(0, cx - rx):cx + rx] = 255
    try:
        got = guide.detect_splines(img, lab)
        ref = dor.detect_splines(img, lab)
    except ValueError as exc:  # e.g. an empty ring: both must raise
        try:
            dor.detect_splines(img, lab)
            print(f"detect it {it}: GPU raised {exc!r}, oracle did not")
            bad += 1
        except ValueError:
            pass
        continue
    g = [(tuple(s.points[0]), tuple(s.points[-1]), tuple(s.direction)) for s in got]
    r = [(tuple(a), tuple(b), tuple(d)) for a, b, d in ref]
    total += len(r)
    if g != r:
        bad += 1
        print(f"detect it {it}: {len(g)} vs {len(r)} splines", g[:2], r[:2], flush=True)
print(f"detection: {n - bad}/{n} ok, {total} splines compared bit for bit")
