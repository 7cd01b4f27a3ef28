"""One tracked fill of a deadlock-regime half-plane (tests/cases.deadlock_scenes),
for ncu captures of the solo shell loop.  python tools/prof_solo.py [case index]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import cases  # noqa: E402
from paper_1611_05319_b200 import FillParams  # noqa: E402
from paper_1611_05319_b200._device import fill_device  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 6
case = cases.deadlock_scenes()[idx]
dev = torch.device("cuda")
img = torch.from_numpy(case["image"][None].astype(np.float32)).to(dev)
lab = torch.from_numpy(case["labels"][None]).to(dev)
g = torch.from_numpy(case["guide"][None]).to(dev)
p = FillParams(**case["params"])
for _ in range(2):
    res = fill_device(img, lab, g, p, tracked=True, rows_cap=1 << 16)
torch.cuda.synchronize()
print(case["name"], res["stats"][0].tolist())
