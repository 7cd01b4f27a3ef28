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


def _ncu_traffic():
    """DRAM bytes of one fill launch from the committed ncu capture (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "round1_ncu_summary.json")) as f:
            return float(json.load(f)["fill_dram_bytes_per_launch"])
    except Exception:
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons polled through NVML during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index=0, period_s=0.002):
        self.index = index
        self.period = period_s
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self._stop.is_set():
                    try:
                        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((mhz, rs))
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=poll, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        mhz = [m for m, _ in self.samples]
        reasons = set()
        for _, rs in self.samples:
            for name, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(mhz)}


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
    # bounded sample: at most ~120 s of CPU work whatever --steps is
    t0 = time.perf_counter()
    done = 0
    while done < args.steps:
        step()
        done += 1
        if time.perf_counter() - t0 > 120.0:
            break
    dt = (time.perf_counter() - t0) / done
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
                         "sample": f"{done} steps x (guide field + full fill of one {sc.name} "
                                   f"frame), numpy restatement of the reference, single-threaded"},
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
    from paper_1611_05319_b200._device import FillGraph, SegmentSet, fill_device

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", torch.cuda.current_device())
    from paper_1611_05319_b200 import scenes

    if args.frames > 1:
        # video batch: this rank's block of C5 frames (seed 1611 + 7919 f)
        batch = [scenes.config("C5", frame=rank * args.frames + i) for i in range(args.frames)]
    else:
        batch = [scene_for(rank, ws, args.config)]
    sc = batch[0]
    params = params_of(sc)
    H, W = sc.labels.shape
    NF = len(batch)
    D = sum(s.n_inpaint for s in batch)

    def to_splines(s):
        return [Spline(id=x["id"], source="user", direction=x["direction"], points=x["points"],
                       kind=x["kind"]) for x in s.splines]

    splines = to_splines(sc)

    # ---- device-resident inputs
    img = torch.from_numpy(np.stack([s.image for s in batch]).astype(np.float32)).to(dev).contiguous()
    lab = torch.from_numpy(np.stack([s.labels for s in batch])).to(dev).contiguous()
    if NF > 1:
        segs = SegmentSet([to_splines(s) for s in batch], dev, per_frame=True)
    else:
        segs = SegmentSet(splines, dev)
    # L2 eviction between steps: write 256 MB, then read another 256 MB so the
    # write-backs of the flush land outside the timed region
    flush_w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_r = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    sink = torch.empty(1, dtype=torch.float32, device=dev)

    def flush_l2():
        flush_w.zero_()
        torch.sum(flush_r, dim=0, keepdim=True, out=sink)
    ws_buf = None

    def step(trace_cap=0):
        # one gf_fill_splines call: the guide field is rastered inside the
        # fill's first pass (same bits as gf_guide_field + gf_fill)
        nonlocal ws_buf
        res = fill_device(img, lab, None, params, tracked=not args.untracked, rows_cap=4096,
                          workspace=ws_buf, splines=segs, trace_cap=trace_cap)
        ws_buf = res["workspace"]
        return res

    for _ in range(max(3, args.warmup)):
        res = step()
    torch.cuda.synchronize()
    # host launch cost of the eager call, measured apart (the graph replay
    # below is what the timed steps run)
    t0 = time.perf_counter()
    for _ in range(20):
        step()
    torch.cuda.synchronize()
    eager_ms = (time.perf_counter() - t0) / 20 * 1e3
    graph = None
    if not args.eager:
        # the whole fill (memset + k_prep + cooperative k_shells) as one CUDA
        # graph: no host launch work per frame (FillGraph, the video path)
        graph = FillGraph(img, lab, None, params, tracked=not args.untracked, rows_cap=4096,
                          splines=segs)
        for _ in range(max(3, args.warmup)):
            res = graph.replay()
        torch.cuda.synchronize()
    stats = res["stats"].cpu().numpy()
    assert int(stats[:, N.STAT_FILLED].sum()) == D, "fill incomplete"
    n_shells = int(stats[:, N.STAT_ITERATIONS].max())

    # per-shell phase trace of one (untimed) step: fill phase, barrier, update
    res = step(trace_cap=256)
    torch.cuda.synchronize()
    trace_all = res["trace"].cpu().numpy()
    tl = trace_all[-1].astype(np.uint64)
    t_start = [int(~np.uint64(tl[2 * i])) for i in range(2)]
    t_end = [int(tl[2 * i + 1]) for i in range(2)]
    timeline = {name: {"start_us": (t_start[i] - t_start[0]) / 1e3,
                       "end_us": (t_end[i] - t_start[0]) / 1e3}
                for i, name in enumerate(["prep", "shells"])}
    tr = trace_all[:n_shells]
    shell_trace = []
    for r in tr:
        row = {"items": int(r[5]), "fill_us": (r[1] - r[0]) / 1e3,
               "lattice_item_max_us": r[6] / 1e3, "rotated_item_max_us": r[7] / 1e3,
               "sync_us": (r[2] - r[1]) / 1e3}
        if args.untracked:
            row.update(rescan_us=(r[3] - r[2]) / 1e3, sync2_us=(r[4] - r[3]) / 1e3)
        shell_trace.append(row)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush_l2()  # evict L2 (126 MB) between steps; not timed
            starts[k].record()
            res = graph.replay() if graph is not None else step()
            ends[k].record()
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_step = sum(step_ms) / len(step_ms)
    t_fill = t_step
    if ws > 1:
        t = torch.tensor([t_step, float(D)], dtype=torch.float64, device=dev)
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dsum = t[1:].clone()
        dist.all_reduce(dsum, op=dist.ReduceOp.SUM)
        t_job, D_job = float(tmax.item()), float(dsum.item())
    else:
        t_job, D_job = t_step, float(D)

    # ---- end-to-end through the public API with host buffers (float64 numpy,
    # the reference's dtype): every step uploads the image and labels and
    # downloads the filled image and the report.  Headline: run_tracked with
    # the splines (rastered inside the fill); also timed: the reference's
    # two-call sequence build_guide_field + run_tracked (field round trip).
    e2e = None
    if not args.no_e2e and NF == 1:
        labels_h = sc.labels
        image_h = sc.image

        def timed(fn, n):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(n):
                fn()
            torch.cuda.synchronize()
            return (time.perf_counter() - t0) / n

        ne = max(3, min(args.steps, 20))
        holder = {}

        def fused():
            holder["u"], _ = tracker.run_tracked(image_h, labels_h, splines, params)

        def dropin():
            fld = build_guide_field(splines, labels_h)
            holder["u2"], _ = tracker.run_tracked(image_h, labels_h, fld, params)
            holder["fld"] = fld

        # the same call on pinned host tensors: the inputs are DMA'd from the
        # caller's pinned memory, the result comes back in a pinned tensor
        image_p = torch.from_numpy(image_h).pin_memory()
        labels_p = torch.from_numpy(labels_h).pin_memory()

        def pinned():
            holder["up"], _ = tracker.run_tracked(image_p, labels_p, splines, params)

        tp = timed(pinned, ne)
        te = timed(fused, ne)
        td = timed(dropin, ne)

        # video from host memory: C5 frames (own masks and splines) in pinned
        # buffers, uploads / fills / downloads pipelined on three streams
        from paper_1611_05319_b200 import video
        from paper_1611_05319_b200.splines import Spline as _Spl
        vframes = [scenes.config("C5", frame=i) for i in range(8)]
        v_img = [torch.from_numpy(f.image).pin_memory() for f in vframes]
        v_lab = [torch.from_numpy(f.labels).pin_memory() for f in vframes]
        v_spl = [[_Spl(id=s_["id"], source="user", direction=s_["direction"],
                       points=s_["points"], kind=s_["kind"]) for s_ in f.splines]
                 for f in vframes]
        v_filled = []

        def consume(f, u, rep):  # a streaming consumer: the result is in host memory
            v_filled.append(rep.filled)

        video.fill_video_host(v_img, v_lab, v_spl, params, on_frame=consume)  # warm-up
        torch.cuda.synchronize()
        v_filled.clear()
        t0 = time.perf_counter()
        video.fill_video_host(v_img + v_img, v_lab + v_lab, v_spl + v_spl, params,
                              on_frame=consume)
        torch.cuda.synchronize()
        tv = (time.perf_counter() - t0) / (2 * len(vframes))
        v_px = sum(v_filled) / len(v_filled)
        u = holder["u"]
        fld = holder["fld"]
        assert np.array_equal(holder["up"].numpy(), u), "pinned path differs from the numpy path"
        delta_px = int((u.view(np.uint64) != np.ascontiguousarray(image_h).view(np.uint64))
                       .any(axis=2).sum())
        e2e = {"value": D / tp / 1e6, "unit": "Mpx/s", "ms_per_frame": tp * 1e3,
               "h2d_bytes_per_step": int(image_h.nbytes + labels_h.nbytes),
               # the result buffer is seeded with the input by D2H DMA as the
               # upload lands, then the changed pixels are written after the fill
               "d2h_bytes_per_step": int(u.nbytes + delta_px * u.shape[2] * u.itemsize),
               "d2h_delta_px": delta_px,
               "path": "tracker.run_tracked(image, labels, splines, params) on pinned host "
                       "tensors (f64 image in, f64 image out, copies in the timed region); "
                       "the result buffer is seeded with the input by D2H DMA while the "
                       "upload runs (gf_upload_mirrored), then gf_output_delta writes the "
                       "changed pixels into it",
               "numpy_ms_per_frame": te * 1e3,
               "numpy_path": "the same call on pageable numpy f64 arrays (the reference's types)",
               "video_pipelined_ms_per_frame": tv * 1e3,
               "video_pipelined_mpx_s": v_px / tv / 1e6,
               "video_path": "video.fill_video_host over 16 C5 frames (8 distinct, own masks and "
                             "splines) in pinned f64 buffers, results streamed to a consumer: "
                             "H2D, fill and D2H of consecutive frames overlap on three streams",
               "dropin_two_call_ms": td * 1e3,
               "dropin_two_call_bytes": int(image_h.nbytes + 2 * labels_h.nbytes + 2 * fld.nbytes
                                            + u.nbytes)}

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    peak, peak_kind = _peaks()
    C = 3
    b_frame = NF * H * W * (C * 4 + C * 4 + 1) + 16 * D  # whole batch
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
            "workload": (f"{sc.name} 1920x1080 disocclusion frame per GPU" if NF == 1 else
                         f"C5 video: {NF} 1080p frames per GPU in one batched launch") +
                        f": guide-field raster + {'untracked' if args.untracked else 'tracked'} "
                        f"shell fill, fp32 RGB in/out, fp64 decisions",
            "global_batch": ws * NF,
            "frames_per_gpu": NF,
            "inpaint_px": D,
            "shells": n_shells,
            "r": sc.params["r"], "mu": sc.params["mu"],
            "ms_per_frame": t_step / NF,
            "ms_step_min": min(step_ms),
            "ms_step_max": max(step_ms),
            "timeline": timeline,
            "shell_trace": shell_trace,
            "l2": "flushed between steps (256 MB write + 256 MB read, untimed)",
            "launch": "CUDA graph replay of memset + k_prep + k_shells" if graph is not None
                      else "eager C-ABI call per step",
            "eager_host_ms_per_call": eager_ms,
            "parallelism": f"frame-parallel x{ws}",
        },
        "roofline": {
            "bound": "hbm",
            "kernel": "gf_fill_splines (k_prep: copy + hull + raster + frontier; k_shells: persistent shell loop + output + Bystander clip)",
            "achieved": achieved,
            "peak": peak,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": _ncu_traffic(),
            "algorithmic_bytes": b_frame,
        },
        "e2e": e2e,
        "gpu_launches": 2 * args.steps,  # k_prep, k_shells
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--untracked", action="store_true")
    ap.add_argument("--frames", type=int, default=1,
                    help="frames per GPU per step (C5 video batch); default 1 = C2 single frame")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time eager calls instead of the CUDA graph")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
