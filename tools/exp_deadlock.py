"""Device time per shell in the deadlock-heavy regime.

    python tools/exp_deadlock.py [--reps 3]

For each half-plane case of tests/cases.deadlock_scenes(): inputs resident on
the device, one gf_fill call per rep timed with CUDA events; prints shells,
guarded fills, ms per fill and us per shell as JSON lines.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import cases  # noqa: E402
from paper_1611_05319_b200 import FillParams  # noqa: E402
from paper_1611_05319_b200 import _native as N  # noqa: E402
from paper_1611_05319_b200._device import fill_device  # noqa: E402


def time_case(case, reps, tracked=True):
    dev = torch.device("cuda")
    img = torch.from_numpy(case["image"][None].astype(np.float32)).to(dev)
    lab = torch.from_numpy(case["labels"][None]).to(dev)
    g = torch.from_numpy(case["guide"][None]).to(dev)
    p = FillParams(**case["params"])
    res = fill_device(img, lab, g, p, tracked=tracked, rows_cap=1 << 16)
    ws = res["workspace"]
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = fill_device(img, lab, g, p, tracked=tracked, rows_cap=1 << 16, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = res["stats"][0].cpu().numpy()
    shells = int(st[N.STAT_ITERATIONS])
    t = min(ts)
    return {"case": case["name"], "tracked": tracked, "shells": shells,
            "guarded": int(st[N.STAT_DEADLOCK]), "filled": int(st[N.STAT_FILLED]),
            "ms": t, "us_per_shell": t * 1e3 / max(1, shells)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--untracked", action="store_true")
    a = ap.parse_args()
    for case in cases.deadlock_scenes():
        print(json.dumps(time_case(case, a.reps, not a.untracked)), flush=True)


if __name__ == "__main__":
    main()
