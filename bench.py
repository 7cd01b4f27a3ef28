"""Benchmark of the B200 Guidefill fill path (BASELINE.json metric).

One step = one pass of the hot path over one synthetic 1920x1080
disocclusion frame (BASELINE.json configs[1] = SURVEY C2: 10 px
object-edge bands, 6 Bezier splines, eps=3, mu=50, smart order, rotated
ghost-pixel balls, tracking on): spline -> guide-field rasteriser, then the
persistent shell-fill kernel with the frontier tracker, then the clipped
output.  Inputs are resident in HBM before the timed region (``value``);
``e2e`` repeats the metric through the public drop-in API with host numpy
buffers (build_guide_field + run_tracked).

Multi-GPU (torchrun): frames are independent, so rank g fills its own frame
(C5 video seed 1611 + 7919 g) with no data-path collective ("weak"
scaling); the only collective is a max-reduction of the timings.

``--impl reference`` times the reference algorithm's CPU implementation
(the numpy port in oracle/, since the Python reference cannot travel to the
GPU box) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpixels inpainted/s and ms per 1080p frame; fill-kernel HBM GB/s vs peak"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def scene_for(rank, ws, config):
    from paper_1611_05319_b200 import scenes

    if ws > 1:
        sc = scenes.config("C5", frame=rank)
        sc.name = "C5"
        return sc
    return scenes.config(config)


def params_of(sc):
    from paper_1611_05319_b200 import FillParams

    return FillParams(**sc.params)


def run_reference(args):
    """CPU baseline: the reference algorithm (numpy port) on the host cores."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import guidefill_oracle as orc

    sc = scene_for(0, 1, args.config)
    p = orc.Params(**sc.params)
    polys = [orc.polyline(s["points"], s["kind"]) for s in sc.splines]
    dirs = [s["direction"] for s in sc.splines]

    def step():
        field = orc.guide_field(polys, dirs, sc.labels)
        orc.fill(sc.image, sc.labels, field, p, tracked=not args.untracked)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    D = sc.n_inpaint
    value = D / dt / 1e6
    line = {
        "metric": METRIC, "value": value, "unit": "Mpx/s", "impl": "reference",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{sc.name} 1920x1080 disocclusion frame, |D|={D}, "
                               f"r={sc.params['r']}, mu={sc.params['mu']}, "
                               f"{'untracked' if args.untracked else 'tracked'}",
                   "global_batch": 1},
        "cpu_baseline": {"value": value, "unit": "Mpx/s", "cores": 1, "kind": "port",
                         "sample": f"guide field + full fill of one {sc.name} frame per step "
                                   f"(numpy restatement of the reference, single-threaded numpy)"},
        "e2e": {"value": value, "unit": "Mpx/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(sc, untracked, max_s=30.0):
    from oracle import guidefill_oracle as orc

    p = orc.Params(**sc.params)
    polys = [orc.polyline(s["points"], s["kind"]) for s in sc.splines]
    dirs = [s["direction"] for s in sc.splines]
    t0 = time.perf_counter()
    field = orc.guide_field(polys, dirs, sc.labels)
    orc.fill(sc.image, sc.labels, field, p, tracked=not untracked)
    dt = time.perf_counter() - t0
    return {"value": sc.n_inpaint / dt / 1e6, "unit": "Mpx/s", "cores": 1, "kind": "port",
            "sample": f"1 x {sc.name} frame (guide field + fill), numpy port of the reference, "
                      f"{dt:.2f} s"}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1611_05319_b200 import Spline, build_guide_field, tracker
    from paper_1611_05319_b200 import _native as N
    from paper_1611_05319_b200._device import SegmentSet, fill_device, guide_field_device

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", torch.cuda.current_device())
    sc = scene_for(rank, ws, args.config)
    params = params_of(sc)
    H, W = sc.labels.shape
    D = sc.n_inpaint
    splines = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
                      kind=s["kind"]) for s in sc.splines]

    # ---- device-resident inputs
    img = torch.from_numpy(sc.image.astype(np.float32)).to(dev).reshape(1, H, W, 3).contiguous()
    lab = torch.from_numpy(sc.labels).to(dev).reshape(1, H, W).contiguous()
    segs = SegmentSet(splines, dev)
    field = torch.empty((1, H, W, 2), dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ws_buf = None

    def step():
        nonlocal ws_buf
        guide_field_device(lab[0], segs, 3.0, out=field[0])
        res = fill_device(img, lab, field, params, tracked=not args.untracked,
                          rows_cap=4096, workspace=ws_buf)
        ws_buf = res["workspace"]
        return res

    for _ in range(max(3, args.warmup)):
        res = step()
    torch.cuda.synchronize()
    stats = res["stats"][0].cpu().numpy()
    assert int(stats[N.STAT_FILLED]) == D, "fill incomplete"
    n_shells = int(stats[N.STAT_ITERATIONS])

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()  # evict L2 (126 MB) between steps; not timed
            starts[k].record()
            guide_field_device(lab[0], segs, 3.0, out=field[0])
            mids[k].record()
            res = fill_device(img, lab, field, params, tracked=not args.untracked,
                              rows_cap=4096, workspace=ws_buf)
            ends[k].record()
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    fill_ms = [m.elapsed_time(e) for m, e in zip(mids, ends)]
    gf_ms = [s.elapsed_time(m) for s, m in zip(starts, mids)]
    t_step = sum(step_ms) / len(step_ms)
    t_fill = sum(fill_ms) / len(fill_ms)
    t_gf = sum(gf_ms) / len(gf_ms)
    if ws > 1:
        t = torch.tensor([t_step, float(D)], dtype=torch.float64, device=dev)
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dsum = t[1:].clone()
        dist.all_reduce(dsum, op=dist.ReduceOp.SUM)
        t_job, D_job = float(tmax.item()), float(dsum.item())
    else:
        t_job, D_job = t_step, float(D)

    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        labels_h = sc.labels
        image_h = sc.image  # float64, the reference API's dtype
        for _ in range(2):
            fld = build_guide_field(splines, labels_h)
            tracker.run_tracked(image_h, labels_h, fld, params)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ne = max(3, min(args.steps, 10))
        for _ in range(ne):
            fld = build_guide_field(splines, labels_h)
            u, wm = tracker.run_tracked(image_h, labels_h, fld, params)
        torch.cuda.synchronize()
        te = (time.perf_counter() - t0) / ne
        h2d = labels_h.nbytes + image_h.nbytes + labels_h.nbytes + fld.nbytes
        d2h = fld.nbytes + u.nbytes
        e2e = {"value": D / te / 1e6, "unit": "Mpx/s", "ms_per_frame": te * 1e3,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "path": "build_guide_field + run_tracked, float64 numpy in/out"}

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    peak, peak_kind = _peaks()
    C = 3
    b_frame = H * W * (C * 4 + C * 4 + 1) + 16 * D
    achieved = b_frame / (t_fill * 1e-3) / 1e9
    cpu = None if (ws > 1 or args.no_cpu) else cpu_baseline(sc, args.untracked)
    line = {
        "metric": METRIC,
        "value": D_job / (t_job * 1e-3) / 1e6,
        "unit": "Mpx/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": t_job,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": f"{sc.name} 1920x1080 disocclusion frame per GPU: guide-field raster + "
                        f"{'untracked' if args.untracked else 'tracked'} shell fill, fp32 RGB "
                        f"in/out, fp64 decisions",
            "global_batch": ws,
            "inpaint_px": D,
            "shells": n_shells,
            "r": sc.params["r"], "mu": sc.params["mu"],
            "ms_per_frame": t_step,
            "ms_fill": t_fill,
            "ms_guide_field": t_gf,
            "l2": "flushed between steps (512 MB write)",
            "parallelism": f"frame-parallel x{ws}",
        },
        "roofline": {
            "bound": "hbm",
            "kernel": "gf_fill (prep + hull + persistent shell loop + finalize)",
            "achieved": achieved,
            "peak": peak,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": None,
            "algorithmic_bytes": b_frame,
        },
        "e2e": e2e,
        "gpu_launches": 7 * args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--untracked", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
