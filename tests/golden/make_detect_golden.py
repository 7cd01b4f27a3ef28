"""Detection fixtures from the REFERENCE package itself (build container only).

    python tests/golden/make_detect_golden.py

For every scene of ``cases.detect_scenes()``: the measurement ring
(guide.compute_ring, guide.py:65-88), the plain and masked structure tensors
at a few ring pixels (guide.py:139-167), make_spline (guide.py:210-267) from
every ring pixel on a sparse grid, and the seed clustering (guide.py:200-207)
of a fixed hit list.  These parts need no Canny, so they run on the reference
with the scikit-image stub.  Writes ``tests/golden/detect_golden.npz``.
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


def main():
    ref = refimport.load()
    guide = ref["guide"]
    out = {}
    for s, (name, img, lab) in enumerate(cases.detect_scenes()):
        key = f"s{s:02d}"
        ring = sorted(guide.compute_ring(lab), key=lambda p: (p[1], p[0]))
        ring = np.array(ring, dtype=np.int64).reshape(-1, 2)
        out[f"{key}_name"] = np.array(name)
        out[f"{key}_ring"] = ring
        pick = ring[:: max(1, len(ring) // 12)][:12]
        tens, mtens, spl = [], [], []
        for i, j in pick:
            tens.append(guide.structure_tensor(img, (i, j)))
            try:
                mtens.append(guide.modified_structure_tensor(img, lab, (i, j)))
            except guide.ZeroMassError:
                mtens.append(np.full((2, 2), np.nan))
            sp = guide.make_spline((i, j), img, lab)
            if sp is None:
                spl.append(np.full(6, np.nan))
            else:
                spl.append(np.concatenate([sp.points.reshape(-1), np.array(sp.direction)]))
        out[f"{key}_pick"] = pick
        out[f"{key}_tensor"] = np.array(tens)
        out[f"{key}_mtensor"] = np.array(mtens)
        out[f"{key}_spline"] = np.array(spl)
        print(name, len(ring), int(np.isnan(np.array(spl)[:, 0]).sum()), "no-entry seeds")
    rng = np.random.default_rng(5)
    hits = [(int(rng.integers(0, 40)), int(rng.integers(0, 40)), float(rng.uniform()))
            for _ in range(200)]
    out["hits"] = np.array(hits)
    out["clustered"] = np.array(guide._cluster_seeds(hits))
    np.savez_compressed(os.path.join(HERE, "detect_golden.npz"), **out)


if __name__ == "__main__":
    main()
