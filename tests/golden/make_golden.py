"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (needs /root/reference):

    python tests/golden/make_golden.py

Writes ``tests/golden/fill_golden.npz`` and ``tests/golden/guide_golden.npz``.
For every case of tests/cases.py it records the reference's output image
bytes, report rows, iteration/deadlock/unfillable counters and the per-shell
frontier/fill sets (through the ``frontier_update`` hook of
engine._fill_loop, engine.py:286/362), encoded as per-pixel enter/fill shell
maps (see oracle/guidefill_oracle.py).  The oracle is checked against these
files by tests/test_oracle_golden.py.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import cases  # noqa: E402
import refimport  # noqa: E402


def run_reference(ref, case):
    engine, tracker, grid = ref["engine"], ref["tracker"], ref["grid"]
    params = engine.FillParams(**case["params"])
    image, labels, guide = case["image"], case["labels"], case["guide"]
    H, W = labels.shape
    if case["tracked"]:
        u, wm = tracker.run_tracked(image, labels, guide, params, debug=True)
        report = wm.report
    else:
        u, report = engine.inpaint(image, labels, guide, params)

    # replay with a recording hook to extract the per-shell sets
    shells = []

    def hook(frontier, fill, filled_idx, lab):
        shells.append((frontier.copy(), fill.copy()))
        nxt = np.flatnonzero(grid.active_boundary_mask(lab, params.periodic_x))
        return int(nxt.size), nxt

    gv = None if guide is None else np.asarray(guide, dtype=np.float64)
    u2, _, rep2 = engine._fill_loop(image, labels, gv, params, hook)
    assert u2.tobytes() == u.tobytes(), case["name"]
    enter = np.full(H * W, -1, dtype=np.int32)
    fillshell = np.full(H * W, -1, dtype=np.int32)
    for k, (fr, fm) in enumerate(shells):
        new = fr[enter[fr] < 0]
        enter[new] = k
        fillshell[fr[fm]] = k
    if report.unfillable:
        stranded = (labels.reshape(-1) == 255) & (fillshell < 0)
        fillshell[stranded] = -2
    rows = np.array(report.rows, dtype=np.int64).reshape(-1, 5)
    stats = np.array([report.iterations, report.filled, report.deadlock_fills,
                      int(report.unfillable), report.unfillable_count], dtype=np.int64)
    return u, rows, stats, enter.reshape(H, W), fillshell.reshape(H, W)


def main():
    ref = refimport.load()
    out = {}
    all_cases = cases.reference_scenes() + cases.random_scenes()
    for idx, case in enumerate(all_cases):
        u, rows, stats, enter, fillshell = run_reference(ref, case)
        key = f"c{idx:03d}"
        out[f"{key}_u"] = u
        out[f"{key}_rows"] = rows
        out[f"{key}_stats"] = stats
        out[f"{key}_enter"] = enter
        out[f"{key}_fillshell"] = fillshell
        out[f"{key}_name"] = np.array(case["name"])
        print(f"{key} {case['name']:40s} iters={stats[0]} filled={stats[1]} "
              f"deadlock={stats[2]} unfillable={stats[3]}")
    np.savez_compressed(os.path.join(HERE, "fill_golden.npz"), **out)

    gout = {}
    Spline = ref["splines"].Spline
    for idx, gc in enumerate(cases.guide_cases()):
        spl = [Spline(id=f"s{k}", source="user", direction=s["direction"], points=s["points"],
                      kind=s["kind"]) for k, s in enumerate(gc["splines"])]
        field = ref["guide"].build_guide_field(spl, gc["labels"], eta=gc["eta"])
        key = f"g{idx:03d}"
        gout[f"{key}_field"] = field
        for k, sp in enumerate(spl):
            gout[f"{key}_poly{k}"] = sp.polyline()
        print(f"{key} splines={len(spl)} nonzero={int(np.count_nonzero(field))}")
    np.savez_compressed(os.path.join(HERE, "guide_golden.npz"), **gout)

    # known-answer values of the reference's own unit tests (test_engine.py:23-139)
    engine, grid = ref["engine"], ref["grid"]
    kat = {}
    H, W = 12, 31
    lab = np.zeros((H, W), dtype=np.uint8)
    lab[6:, :] = 255
    img = np.zeros((H, W, 1))
    img[:6, :, 0] = 0.8
    import math
    th = math.radians(10.0)
    g10 = (math.cos(th), math.sin(th))
    kat["conf_flat"] = engine.confidence((15, 6), img, lab, (0.0, 1.0), engine.FillParams())
    kat["conf_rot10"] = engine.confidence((15, 6), img, lab, g10, engine.FillParams())
    kat["conf_axis10"] = engine.confidence((15, 6), img, lab, g10,
                                           engine.FillParams(neighborhood="axis_ball"))
    lab1 = np.full((1, 7), 255, dtype=np.uint8)
    lab1[0, :3] = 0
    img1 = np.zeros((1, 7, 1))
    img1[0, :3, 0] = [0.0, 0.3, 0.9]
    kat["fill_muinf"] = engine.fill_color((3, 0), img1, lab1, (1.0, 0.0),
                                          engine.FillParams(mu=math.inf))[0][0]
    for k, v in kat.items():
        print(k, repr(float(v)))
    np.savez(os.path.join(HERE, "kat_golden.npz"), **{k: np.float64(v) for k, v in kat.items()})


if __name__ == "__main__":
    main()
