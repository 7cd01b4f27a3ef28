"""Experiment: per-phase maxima of one work unit per shell (needs a -DGF_FINE_TRACE build,
selected with GF_B200_LIB)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, Spline, FillParams
from paper_1611_05319_b200._device import fill_device, SegmentSet

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
sc = scenes.config(cfg)
dev = torch.device("cuda")
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in sc.splines]
img = torch.from_numpy(sc.image.astype(np.float32))[None].to(dev).contiguous()
lab = torch.from_numpy(sc.labels)[None].to(dev).contiguous()
segs = SegmentSet(spl, dev)
p = FillParams(**sc.params)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for rep in range(4):
    flush.zero_()
    res = fill_device(img, lab, None, p, splines=segs, trace_cap=256, rows_cap=4096)
    torch.cuda.synchronize()
t = res["trace"].cpu().numpy()
n = int(res["stats"][0, 0].item())
print(f"{cfg}: shells {n}")
print("k  items  fill  sync | entry_max eval_max eval_mean n | fetch rest | decide activate  (means, us)")
for k in range(n):
    r, f = t[k], t[128 + k]
    c = max(1, f[3])
    print(f"{k:2d} {r[5]:6d} {(r[1]-r[0])/1e3:5.2f} {(r[2]-r[1])/1e3:5.2f} | "
          f"{f[0]/1e3:5.2f} {f[1]/1e3:5.2f} {f[2]/c/1e3:5.2f} {f[3]:6d} | {f[4]/c/1e3:5.2f} {f[5]/c/1e3:5.2f} | {f[6]/c/1e3:5.2f} {f[7]/c/1e3:5.2f}")
