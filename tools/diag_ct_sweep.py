"""Which random coherence scene makes the persistent loop and the shell loop differ."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import cases  # noqa: E402
from oracle import guidefill_oracle as orc  # noqa: E402
from paper_1611_05319_b200 import FillParams  # noqa: E402
from paper_1611_05319_b200.coherence import run_coherence_fill, run_coherence_fill_shells  # noqa: E402

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
    d_img = torch.from_numpy(img).cuda()
    d_lab = torch.from_numpy(lab).cuda()
    a = run_coherence_fill(d_img.clone(), d_lab, p, tracked, True)
    b = run_coherence_fill(d_img.clone(), d_lab, p, tracked, True)
    c = run_coherence_fill_shells(d_img.clone(), d_lab, p, tracked, True)
    ua, ub, uc = (x[0].cpu().numpy() for x in (a, b, c))
    same_ab = np.array_equal(ua.view(np.int64), ub.view(np.int64))
    same_ac = np.array_equal(ua.view(np.int64), uc.view(np.int64))
    if not (same_ab and same_ac):
        ref = orc.fill(img, lab, None, orc.Params.of(p), tracked=tracked)
        ur = ref["u"]
        d = np.argwhere(ua != uc)
        print(f"it {it} {p} tracked={tracked} C={C} HxW={H}x{W}: ab {same_ab} ac {same_ac}; "
              f"persistent==oracle {np.array_equal(ua, ur)} shells==oracle {np.array_equal(uc, ur)}; "
              f"{len(d)} diffs, first {d[:3].tolist()}, rep unfillable {a[1]['unfillable']} {c[1]['unfillable']}",
              flush=True)
        j, i = d[0][:2]
        print("   lab at", lab[j, i], "fillshell", a[3].reshape(H, W)[j, i].item(), c[3].reshape(H, W)[j, i].item(),
              "vals", ua[j, i], uc[j, i], ur[j, i])
print("done")
