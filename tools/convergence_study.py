"""Convergence of the GPU fill to its continuum transport limit (PAPER.md
Section 4; the reference's limits.convergence_study) past the reference's
1024 px: dyadic strips up to 8192 x 8197 (67 M px, 8192 onion shells).
Usage: python tools/convergence_study.py [out.json]
"""
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_05319_b200 import limits  # noqa: E402

RES = (128, 256, 512, 1024, 2048, 4096, 8192)


def main():
    traces = {"smooth_sin": lambda x: np.sin(2.0 * np.pi * np.asarray(x)),
              "step": lambda x: np.where(np.mod(np.asarray(x), 1.0) < 0.5, 0.0, 1.0)}
    out = {}
    for name, tr in traces.items():
        for kind, g in (("rotated_ball", (0.0, 1.0)), ("rotated_ball", (0.5, 0.8)),
                        ("axis_ball", (0.5, 0.8))):
            t0 = time.perf_counter()
            st = limits.convergence_study(tr, kind=kind, r=3, mu=1.0, g=g, resolutions=RES)
            key = f"{name}/{kind}/g=({g[0]},{g[1]})"
            out[key] = {"theta_star_deg": math.degrees(st["theta_star_rad"]),
                        "errors": {str(n): {str(p): e for p, e in st["errors"][n].items()}
                                   for n in RES},
                        "orders": {str(p): o for p, o in st["orders"].items()},
                        "wall_s": time.perf_counter() - t0}
            print(key, "theta* %.3f deg" % out[key]["theta_star_deg"],
                  "Linf orders", [None if o is None else round(o, 3) for o in st["orders"][math.inf]],
                  "L1 orders", [None if o is None else round(o, 3) for o in st["orders"][1]],
                  "%.1f s" % out[key]["wall_s"], flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
