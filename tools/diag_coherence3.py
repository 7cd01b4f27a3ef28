"""Per shell of a coherence case: the GPU frontier (query points) against the
oracle's, and the deadlock pick on each side."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases  # noqa: E402
from oracle import guidefill_oracle as orc  # noqa: E402
from paper_1611_05319_b200 import FillParams, coherence, engine  # noqa: E402

CT = cases.coherence_scenes()
orig_sp = coherence.sample_points_device
orig_of = orc.sample_frontier
dev, ora = [], []


def wrapped_sp(u, lab, pts, g, params):
    rw, tw, vals = orig_sp(u, lab, pts, g, params)
    dev.append((pts.cpu().numpy().copy(), (rw / tw).cpu().numpy(), g.cpu().numpy().copy(), rw.cpu().numpy(), tw.cpu().numpy()))
    return rw, tw, vals


def wrapped_of(u, readable, fx, fy, g, params, offs):
    v, rw, tw = orig_of(u, readable, fx, fy, g, params, offs)
    ora.append((np.stack([fx, fy], 1).copy(), rw / tw, np.array(g, copy=True), rw, tw))
    return v, rw, tw


coherence.sample_points_device = wrapped_sp
orc.sample_frontier = wrapped_of
for idx in [int(a) for a in sys.argv[1:]] or (12, 15):
    dev.clear()
    ora.clear()
    case = CT[idx]
    p = FillParams(**case["params"])
    engine._run_fill(case["image"], case["labels"], None, p, tracked=case["tracked"], order_log=True)
    orc.fill(case["image"], case["labels"], None, orc.Params.of(p), tracked=case["tracked"])
    print("case", idx, case["name"], "shells", len(dev), len(ora))
    for k, ((pd, cd, gd, rwd, twd), (po, co, go, rwo, two)) in enumerate(zip(dev, ora)):
        same_pts = pd.shape == po.shape and np.array_equal(pd, po)
        same_c = same_pts and np.array_equal(cd.view(np.int64), co.view(np.int64))
        if not (same_pts and same_c):
            print(f" shell {k}: same frontier {same_pts} ({len(pd)} vs {len(po)}), same conf {same_c}")
            if same_pts:
                bad = np.flatnonzero(cd.view(np.int64) != co.view(np.int64))
                print("   conf diffs at", bad[:5], cd[bad[:5]], co[bad[:5]])
                for i in bad[:3]:
                    print("   i", i, "g dev", [hex(v) for v in gd[i].view(np.uint64)], "g ora",
                          [hex(v) for v in go[i].view(np.uint64)], "rw", rwd[i], rwo[i], "tw", twd[i], two[i])
            else:
                sd = set(map(tuple, pd.tolist()))
                so = set(map(tuple, po.tolist()))
                print("   only dev", sorted(sd - so)[:5], "only oracle", sorted(so - sd)[:5])
                if sd == so:
                    print("   same set, different order; dev argmax", pd[int(np.argmax(cd))],
                          "oracle argmax", po[int(np.argmax(co))])
            break
