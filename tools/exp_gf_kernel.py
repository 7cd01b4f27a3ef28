"""Experiment: dense guide-field kernel time (C2, C4) with CUDA events."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, Spline
from paper_1611_05319_b200._device import SegmentSet, guide_field_device
for name in ("C2", "C4"):
    sc = scenes.config(name); dev = torch.device("cuda")
    spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in sc.splines]
    segs = SegmentSet(spl, dev); d_lab = torch.from_numpy(sc.labels).to(dev)
    out = guide_field_device(d_lab, segs, 3.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): guide_field_device(d_lab, segs, 3.0, out=out)
    e1.record(); torch.cuda.synchronize()
    print(name, "n_seg", segs.n_seg, "inpaint", int((sc.labels == 255).sum()), "kernel ms %.4f" % (e0.elapsed_time(e1) / 20), flush=True)
