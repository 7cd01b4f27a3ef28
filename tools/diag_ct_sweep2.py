"""Shell loop vs oracle on sweep scene 13: per shell, g and rw/tw of the shell loop's
kernels against the oracle's on the same state."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases  # noqa: E402
from oracle import guidefill_oracle as orc  # noqa: E402
from paper_1611_05319_b200 import FillParams, coherence  # noqa: E402

target = int(sys.argv[1]) if len(sys.argv) > 1 else 13
rng = np.random.default_rng(31337)
for it in range(40):
    lab = cases.islands_labels(rng, 24, 90)
    H, W = lab.shape
    C = int(rng.integers(1, 5))
    img = rng.uniform(size=(H, W, C))
    img[lab == 255] = 0.0
    order = ["onion", "smart", "smart_with_data_term"][it % 3]
    p = FillParams(r=int(rng.integers(1, 7)), mu=float(rng.choice([0.0, 10.0, 50.0, math.inf])),
                   order=order, c2=float(rng.uniform(0.1, 0.8)),
                   neighborhood=["rotated_ball", "axis_ball"][it % 2],
                   g_source="modified_structure_tensor", periodic_x=bool(it % 5 == 0),
                   sigma=float(rng.choice([1.0, 2.0, 2.5])), rho=float(rng.choice([2.0, 4.0])))
    tracked = bool(it % 4 != 3)
    if it == target:
        break
orig_g = coherence.coherence_directions_device
orig_sp = coherence.sample_points_device
state = {"k": 0}


def g_hook(u, lab_, idx, sigma, rho, lam, ws, pts):
    g = orig_g(u, lab_, idx, sigma, rho, lam, ws, pts)
    f = idx.cpu().numpy()
    iy, ix = np.divmod(f, W)
    go = orc.coherence_directions(u.cpu().numpy(), lab_.cpu().numpy() == 0, ix, iy, sigma, rho, lam)
    gd = g.cpu().numpy()
    bad = np.flatnonzero(np.any(gd.view(np.int64) != go.view(np.int64), axis=1))
    if bad.size:
        i = bad[0]
        print(f"shell {state['k']}: g differs at {bad.size} of {len(f)}; first px ({ix[i]}, {iy[i]}) "
              f"dev {gd[i].tolist()} oracle {go[i].tolist()}")
    return g


def sp_hook(u, lab_, pts, g, params):
    rw, tw, vals = orig_sp(u, lab_, pts, g, params)
    P = pts.cpu().numpy()
    op = orc.Params.of(params)
    v_o, rw_o, tw_o = orc.sample_frontier(u.cpu().numpy(), lab_.cpu().numpy() == 0, P[:, 0].copy(),
                                          P[:, 1].copy(), g.cpu().numpy(), op,
                                          orc.disk_offsets(op.r)[1:])
    vd = vals.cpu().numpy()
    bad = np.flatnonzero(np.any(vd.view(np.int64) != v_o.view(np.int64), axis=1) |
                         (rw.cpu().numpy() != rw_o) | (tw.cpu().numpy() != tw_o))
    if bad.size:
        i = bad[0]
        print(f"shell {state['k']}: sample differs at {bad.size}; first pt {P[i].tolist()} rw {rw[i].item()} "
              f"{rw_o[i]} vals {vd[i].tolist()} {v_o[i].tolist()}")
    state["k"] += 1
    return rw, tw, vals


coherence.coherence_directions_device = g_hook
coherence.sample_points_device = sp_hook
print(p, tracked, H, W, C)
coherence.run_coherence_fill_shells(torch.from_numpy(img).cuda(), torch.from_numpy(lab).cuda(), p,
                                    tracked, True)
print("done")

# final values: shell loop vs persistent vs oracle, in bits, and the hull
from paper_1611_05319_b200.coherence import run_coherence_fill  # noqa: E402
coherence.coherence_directions_device = orig_g
coherence.sample_points_device = orig_sp
a = run_coherence_fill(torch.from_numpy(img).cuda(), torch.from_numpy(lab).cuda(), p, tracked, True)
c = coherence.run_coherence_fill_shells(torch.from_numpy(img).cuda(), torch.from_numpy(lab).cuda(), p,
                                        tracked, True)
ref = orc.fill(img, lab, None, orc.Params.of(p), tracked=tracked)
ua, uc, ur = a[0].cpu().numpy(), c[0].cpu().numpy(), ref["u"]
rd = img[lab == 0]
print("hull", rd.min().hex(), rd.max().hex())
for j, i, ch in np.argwhere(ua != uc)[:4]:
    print((j, i, ch), "persistent", ua[j, i, ch].hex(), "shells", uc[j, i, ch].hex(), "oracle",
          ur[j, i, ch].hex(), "deadlock fills", a[1]["deadlock_fills"], c[1]["deadlock_fills"])
