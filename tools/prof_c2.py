"""C2 fill (f32 device frames, splines fused) run a few times: ncu target."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import numpy as np, torch
from paper_1611_05319_b200 import FillParams, Spline, scenes
from paper_1611_05319_b200._device import SegmentSet, fill_device
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
sc = scenes.config(name)
dev = torch.device("cuda")
img = torch.from_numpy(sc.image[None].astype(np.float32)).to(dev)
lab = torch.from_numpy(sc.labels[None]).to(dev)
segs = SegmentSet([Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
                          kind=s["kind"]) for s in sc.splines], dev)
p = FillParams(**sc.params)
ws = None
for _ in range(3):
    r = fill_device(img, lab, None, p, splines=segs, workspace=ws, rows_cap=4096)
    ws = r["workspace"]
torch.cuda.synchronize()
print(name, r["stats"][0].tolist())
