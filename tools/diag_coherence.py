"""Diagnose GPU-vs-reference order differences on the smart-order coherence cases:
per shell, max |g_device - g_oracle| on the same state and, on deadlock shells,
the gap between the two largest confidences."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases  # noqa: E402
from oracle import guidefill_oracle as orc  # noqa: E402
from paper_1611_05319_b200 import FillParams, coherence, engine  # noqa: E402

gold = np.load(os.path.join(ROOT, "tests/golden/coherence_golden.npz"))
CT = cases.coherence_scenes()
orig = coherence.coherence_directions_device
orig_sp = coherence.sample_points_device
log = []


def wrapped(u, lab, idx, sigma=2.0, rho=4.0, lam=1e-5, workspace=None, points=None):
    g = orig(u, lab, idx, sigma, rho, lam, workspace, points)
    W = lab.shape[1]
    f = idx.cpu().numpy()
    iy, ix = np.divmod(f, W)
    go = orc.coherence_directions(u.cpu().numpy(), lab.cpu().numpy() == 0, ix, iy, sigma, rho, lam)
    log.append(dict(dg=float(np.abs(g.cpu().numpy() - go).max())))
    return g


def wrapped_sp(u, lab, pts, g, params):
    rw, tw, vals = orig_sp(u, lab, pts, g, params)
    conf = (rw / tw).cpu().numpy()
    srt = np.sort(conf[np.isfinite(conf)])[::-1]
    log[-1].update(top2=(srt[:2].tolist() if srt.size else []),
                   near_c=float(np.min(np.abs(conf - params.c))) if conf.size else None)
    return rw, tw, vals


coherence.coherence_directions_device = wrapped
coherence.sample_points_device = wrapped_sp
for idx in [int(a) for a in sys.argv[1:]] or (11, 12):
    log.clear()
    case = CT[idx]
    p = FillParams(**case["params"])
    u, rep, maps = engine._run_fill(case["image"], case["labels"], None, p, tracked=case["tracked"],
                                    order_log=True)
    gf = gold[f"c{idx:03d}_fillshell"]
    diff = np.argwhere(maps["fillshell"] != gf)
    first = min(int(min(maps["fillshell"][tuple(d)], gf[tuple(d)])) for d in diff) if len(diff) else None
    print(f"case {idx} {case['name']}: {len(diff)} px differ, first differing shell {first}")
    for k, e in enumerate(log[: (first or 0) + 2]):
        print(k, e)
