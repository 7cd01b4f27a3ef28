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


def trace_case(case, tracked=True, cap=32768):
    """Per-shell globaltimer trace of one fill: shell start-to-start gaps and
    the fill-phase span (slot 1 - slot 0)."""
    dev = torch.device("cuda")
    img = torch.from_numpy(case["image"][None].astype(np.float32)).to(dev)
    lab = torch.from_numpy(case["labels"][None]).to(dev)
    g = torch.from_numpy(case["guide"][None]).to(dev)
    p = FillParams(**case["params"])
    res = fill_device(img, lab, g, p, tracked=tracked, rows_cap=1 << 16, trace_cap=cap)
    torch.cuda.synchronize()
    tr = res["trace"].cpu().numpy().astype(np.int64)
    n = min(int(res["stats"][0, N.STAT_ITERATIONS]), cap - 1)
    st = tr[:n, 0]
    gaps = np.diff(st) / 1e3
    span = (tr[:n, 1] - tr[:n, 0]) / 1e3
    rows = res["rows"][0, :n].cpu().numpy()
    one = rows[:-1, 1] == 1
    # solo shells: phase marks in slots 2 (eval), 3 (decide), 4 (fills),
    # 6 (activation), 7 (booking), 1 (end)
    ph = {}
    solo = tr[:n, 7] > 0
    if solo.any():
        t = tr[:n][solo]
        for name, a, b in (("dirty", 0, 2), ("eval", 2, 3), ("decide_guard", 3, 4),
                           ("fills_6a", 4, 6), ("activate", 6, 7), ("book", 7, 1)):
            ph[name] = float(np.median((t[:, b] - t[:, a]) / 1e3))
    return {"case": case["name"], "shells_traced": n, "solo_shells": int(solo.sum()),
            "solo_phase_us_median": ph,
            "gap_us_median": float(np.median(gaps)), "gap_us_p90": float(np.percentile(gaps, 90)),
            "gap_us_one_fill_median": float(np.median(gaps[one])) if one.any() else None,
            "span_us_median": float(np.median(span)),
            "gap_hist": np.histogram(gaps, bins=[0, 2, 4, 6, 8, 12, 16, 24, 32, 64, 1e9])[0].tolist()}


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
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--grid", action="store_true", help="force the grid loop (GF_SOLO=0)")
    a = ap.parse_args()
    if a.grid:
        os.environ["GF_SOLO"] = "0"
    if a.trace:
        for case in cases.deadlock_scenes(mus=(50.0,)):
            print(json.dumps(trace_case(case, not a.untracked)), flush=True)
        return
    for case in cases.deadlock_scenes():
        print(json.dumps(time_case(case, a.reps, not a.untracked)), flush=True)


if __name__ == "__main__":
    main()
