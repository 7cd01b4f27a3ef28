"""Coherence-transport preset on the C2 frame (1920x1080, 77,440 Inpaint px):
GPU shell-by-shell loop vs the CPU oracle (numpy/scipy restatement of the
reference), order bit-exactness and max |du| on the full frame."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
from oracle import guidefill_oracle as orc  # noqa: E402
from paper_1611_05319_b200 import FillParams, engine, scenes  # noqa: E402
from paper_1611_05319_b200.coherence import run_coherence_fill  # noqa: E402

sc = scenes.config("C2")
p = FillParams.coherence_transport()
H, W = sc.labels.shape
d_img = torch.from_numpy(np.ascontiguousarray(sc.image, dtype=np.float64)).cuda()
d_lab = torch.from_numpy(sc.labels).cuda()
for _ in range(2):
    run_coherence_fill(d_img.clone(), d_lab, p, tracked=True)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    u0 = d_img.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, rep, _, _ = run_coherence_fill(u0, d_lab, p, tracked=True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
# kernel share: one structure-tensor evaluation over the frame
from paper_1611_05319_b200.coherence import coherence_directions_device  # noqa: E402
idx = torch.nonzero(d_lab.reshape(-1) == 255).reshape(-1)[:14000]
for _ in range(3):
    coherence_directions_device(d_img, d_lab, idx)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    coherence_directions_device(d_img, d_lab, idx)
e1.record()
torch.cuda.synchronize()
ct_ms = e0.elapsed_time(e1) / 20
u, rep2, maps = engine._run_fill(sc.image, sc.labels, None, p, tracked=True, order_log=True)
t0 = time.perf_counter()
ref = orc.fill(sc.image, sc.labels, None, orc.Params.of(p), tracked=True)
cpu_s = time.perf_counter() - t0
res = dict(workload="C2 frame, FillParams.coherence_transport() (r=5, axis ball, onion, g from the "
           "masked structure tensor, sigma 2, rho 4)", shells=rep["iterations"], filled=rep["filled"],
           gpu_ms_per_frame_device_resident=min(ts), gpu_ms_all=ts,
           tensor_eval_ms=ct_ms, tensor_evals_per_frame=rep["iterations"],
           order_bit_exact=bool(np.array_equal(maps["fillshell"], ref["fillshell"])
                                and np.array_equal(maps["enter"], ref["enter"])),
           rows_equal=[tuple(r) for r in rep2.rows] == [tuple(r) for r in ref["rows"]],
           max_abs_du=float(np.abs(u - ref["u"]).max()),
           cpu_oracle_s=cpu_s, cpu_cores=1,
           mpx_s_gpu=rep["filled"] / (min(ts) * 1e3), mpx_s_cpu=rep["filled"] / (cpu_s * 1e6))
print(json.dumps(res))
