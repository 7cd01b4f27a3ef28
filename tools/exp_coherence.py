"""Coherence-transport preset on the C2 frame (1920x1080, 77,440 Inpaint px):
the persistent-kernel loop (run_coherence_fill) and the shell-by-shell loop
(run_coherence_fill_shells) vs the CPU oracle (numpy/scipy restatement of the
reference): time per frame, order bit-exactness and max |du| on the full frame."""
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
from paper_1611_05319_b200.coherence import (run_coherence_fill,  # noqa: E402
                                             run_coherence_fill_shells)

sc = scenes.config("C2")
p = FillParams.coherence_transport()
H, W = sc.labels.shape
d_img = torch.from_numpy(np.ascontiguousarray(sc.image, dtype=np.float64)).cuda()
d_lab = torch.from_numpy(sc.labels).cuda()


def timed(fn, reps=7):
    for _ in range(2):
        fn(d_img.clone(), d_lab, p, tracked=True)
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        u0 = d_img.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        uu, rr, _, fs = fn(u0, d_lab, p, tracked=True)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return out, uu, rr, fs


ts, u_k, rep, fs_k = timed(run_coherence_fill)
ts_sh, u_s, rep_sh, fs_s = timed(run_coherence_fill_shells, 3)
same_paths = bool(torch.equal(fs_k, fs_s) and torch.equal(u_k.view(torch.int64), u_s.view(torch.int64))
                  and rep["rows"] == rep_sh["rows"])
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
           path="run_coherence_fill: one persistent cooperative kernel (gf_coherence_fill)",
           shells_path_ms=min(ts_sh), shells_path_ms_all=ts_sh,
           persistent_equals_shells_path_bitwise=same_paths,
           tensor_eval_ms=ct_ms, tensor_evals_per_frame=rep["iterations"],
           order_bit_exact=bool(np.array_equal(maps["fillshell"], ref["fillshell"])
                                and np.array_equal(maps["enter"], ref["enter"])),
           rows_equal=[tuple(r) for r in rep2.rows] == [tuple(r) for r in ref["rows"]],
           max_abs_du=float(np.abs(u - ref["u"]).max()),
           cpu_oracle_s=cpu_s, cpu_cores=1,
           mpx_s_gpu=rep["filled"] / (min(ts) * 1e3), mpx_s_cpu=rep["filled"] / (cpu_s * 1e6))
print(json.dumps(res))
