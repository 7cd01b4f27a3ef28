"""Coherence-transport fixtures from the REFERENCE package itself (build container only).

    python tests/golden/make_coherence_golden.py

Writes ``tests/golden/coherence_golden.npz``: for every case of
``cases.coherence_scenes()`` the reference's output image, report rows,
counters and per-shell enter/fill maps (same encoding as make_golden.py), and
``guide.coherence_directions`` (guide.py:330-355) at every Inpaint pixel of
``cases.edge_block()``.
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
from make_golden import run_reference  # noqa: E402


def main():
    ref = refimport.load()
    out = {}
    for idx, case in enumerate(cases.coherence_scenes()):
        u, rows, stats, enter, fillshell = run_reference(ref, case)
        key = f"c{idx:03d}"
        out[f"{key}_u"] = u
        out[f"{key}_rows"] = rows
        out[f"{key}_stats"] = stats
        out[f"{key}_enter"] = enter
        out[f"{key}_fillshell"] = fillshell
        out[f"{key}_name"] = np.array(case["name"])
        print(case["name"], stats.tolist())
    img, lab = cases.edge_block()
    jj, ii = np.nonzero(lab == 255)
    for s, r in ((2.0, 4.0), (1.0, 2.0)):
        g = ref["guide"].coherence_directions(img, lab == 0, ii, jj, sigma=s, rho=r)
        out[f"dirs_s{s:g}_r{r:g}"] = g
    out["dirs_ii"] = ii
    out["dirs_jj"] = jj
    np.savez_compressed(os.path.join(HERE, "coherence_golden.npz"), **out)


if __name__ == "__main__":
    main()
