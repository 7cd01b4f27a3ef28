"""Experiment: prep/shell/finalize timeline under different guide sources."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, Spline, FillParams, build_guide_field
from paper_1611_05319_b200._device import fill_device, SegmentSet

sc = scenes.config("C2")
dev = torch.device("cuda")
H, W = sc.labels.shape
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in sc.splines]
img = torch.from_numpy(sc.image.astype(np.float32))[None].to(dev).contiguous()
lab = torch.from_numpy(sc.labels)[None].to(dev).contiguous()
field = torch.from_numpy(build_guide_field(spl, sc.labels))[None].to(dev).contiguous()
segs = SegmentSet(spl, dev)
p = FillParams(**sc.params)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)

def tl(res):
    t = res["trace"].cpu().numpy()[-1].astype(np.uint64)
    s = [int(~np.uint64(t[2 * i])) for i in range(3)]
    e = [int(t[2 * i + 1]) for i in range(3)]
    return [round((e[i] - s[i]) / 1e3, 1) for i in range(3)]

for name, kw in [("raster", dict(guide=None, splines=segs)), ("field", dict(guide=field)),
                 ("none", dict(guide=None))]:
    out = []
    for rep in range(5):
        flush.zero_()
        res = fill_device(img, lab, kw.get("guide"), p, splines=kw.get("splines"), trace_cap=64, rows_cap=4096)
        torch.cuda.synchronize()
        out.append(tl(res))
    print(name, "prep/shells/finalize us:", out[-3:])
# label-only scene: no inpaint at all
lab0 = torch.zeros_like(lab)
for rep in range(3):
    flush.zero_()
    res = fill_device(img, lab0, None, p, trace_cap=64, rows_cap=16)
    torch.cuda.synchronize()
print("no-D frame prep/shells/finalize us:", tl(res))
