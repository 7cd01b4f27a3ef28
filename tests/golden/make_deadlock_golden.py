"""Deadlock-regime fixtures from the REFERENCE package itself (build container only).

    python tests/golden/make_deadlock_golden.py

For every case of ``cases.deadlock_scenes()`` (256x256 half-planes, rotated
guide at 10/25/40/73 degrees, smart order, mu 50/100: SURVEY.md Appendix B)
one run of the reference's ``engine._fill_loop`` (engine.py:286-376) with a
recording ``frontier_update`` hook (engine.py:362) that returns the
reference's own full rescan (grid.active_boundary_mask) -- the sets the
tracker provably yields (tracker.py:161-168).
Writes ``tests/golden/deadlock_golden.npz``: output values at the Inpaint
pixels (16-bit quantised), per-shell
(frontier size, filled) rows, counters and the per-pixel enter/fill shell
maps.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import cases  # noqa: E402
import refimport  # noqa: E402


def run(ref, case):
    engine, grid = ref["engine"], ref["grid"]
    params = engine.FillParams(**case["params"])
    labels = case["labels"]
    H, W = labels.shape
    enter = np.full(H * W, -1, dtype=np.int32)
    fillshell = np.full(H * W, -1, dtype=np.int32)
    k = [0]

    def hook(frontier, fill, filled_idx, lab):
        new = frontier[enter[frontier] < 0]
        enter[new] = k[0]
        fillshell[frontier[fill]] = k[0]
        k[0] += 1
        nxt = np.flatnonzero(grid.active_boundary_mask(lab, params.periodic_x))
        return int(nxt.size), nxt

    u, _, rep = engine._fill_loop(case["image"], labels, case["guide"], params, hook)
    rows = np.array([(r[1], r[4]) for r in rep.rows], dtype=np.int32).reshape(-1, 2)
    stats = np.array([rep.iterations, rep.filled, rep.deadlock_fills, int(rep.unfillable),
                      rep.unfillable_count], dtype=np.int64)
    return u, rows, stats, enter.reshape(H, W), fillshell.reshape(H, W)


def main():
    ref = refimport.load()
    out = {}
    for idx, case in enumerate(cases.deadlock_scenes()):
        t0 = time.perf_counter()
        u, rows, stats, enter, fillshell = run(ref, case)
        key = f"d{idx:03d}"
        # Inpaint pixels only (the rest is the input), quantised to 16 bits:
        # |error| <= 7.7e-6, far inside the 1e-4 value tolerance
        out[f"{key}_uq"] = np.round(u[case["labels"] == 255] * 65535).astype(np.uint16)
        out[f"{key}_rows"] = rows
        out[f"{key}_stats"] = stats
        out[f"{key}_enter"] = enter
        out[f"{key}_fillshell"] = fillshell
        out[f"{key}_name"] = np.array(case["name"])
        print(case["name"], stats.tolist(), f"{time.perf_counter() - t0:.1f} s", flush=True)
    np.savez_compressed(os.path.join(HERE, "deadlock_golden.npz"), **out)


if __name__ == "__main__":
    main()
