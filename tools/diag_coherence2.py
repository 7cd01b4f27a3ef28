"""Per shell of a coherence case: GPU rw / tw (sample_points_device) against the
oracle's sample_frontier on the same state, frontier and g (bitwise)."""
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
state = {}


def wrapped_sp(u, lab, pts, g, params):
    rw, tw, vals = orig_sp(u, lab, pts, g, params)
    un, ln = u.cpu().numpy(), lab.cpu().numpy()
    P = pts.cpu().numpy()
    gn = g.cpu().numpy()
    op = orc.Params.of(params)
    offs = orc.disk_offsets(op.r)[1:]
    v_o, rw_o, tw_o = orc.sample_frontier(un, ln == 0, P[:, 0].copy(), P[:, 1].copy(), gn, op, offs)
    rw_d, tw_d = rw.cpu().numpy(), tw.cpu().numpy()
    brw = np.flatnonzero(rw_d.view(np.int64) != rw_o.view(np.int64))
    btw = np.flatnonzero(tw_d.view(np.int64) != tw_o.view(np.int64))
    k = state.setdefault("k", 0)
    state["k"] = k + 1
    if brw.size or btw.size:
        i = int(brw[0]) if brw.size else int(btw[0])
        print(f"shell {k}: F={rw_d.size} rw mismatches {brw.size}, tw mismatches {btw.size}; first i={i}"
              f" rw {rw_d[i]!r} vs {rw_o[i]!r}, tw {tw_d[i]!r} vs {tw_o[i]!r}, g {gn[i].tolist()},"
              f" pt {P[i].tolist()}")
        state.setdefault("bad", (i, P[i].copy(), gn[i].copy()))
    return rw, tw, vals


coherence.sample_points_device = wrapped_sp
for idx in [int(a) for a in sys.argv[1:]] or (12, 15):
    state.clear()
    case = CT[idx]
    p = FillParams(**case["params"])
    print("case", idx, case["name"], case["params"])
    engine._run_fill(case["image"], case["labels"], None, p, tracked=case["tracked"], order_log=True)
    if "bad" in state:
        i, pt, g = state["bad"]
        op = orc.Params.of(p)
        offs = orc.disk_offsets(op.r)[1:]
        rel = orc.ball_points(g[None, :], offs, True)[0]
        w = orc.ball_weights(rel, g[None, :], op.mu, op.r)
        print("g bits", [hex(v) for v in g.view(np.uint64)], "weights", w.ravel()[:8].tolist())
