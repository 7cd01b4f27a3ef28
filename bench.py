"""Benchmark of the B200 Guidefill fill path (BASELINE.json metric).

Workloads:

* C2 (BASELINE.json configs[1]) -- one synthetic 1920x1080 disocclusion
  frame: 10 px object-edge bands, 6 Bezier splines, eps=3, mu=50, smart
  order, rotated ghost-pixel balls, tracking on.  One step = spline ->
  guide-field raster, the persistent shell-fill kernel with the frontier
  tracker, the clipped output.  This is ``value`` at N = 1.
* C5 (configs[4]) -- the 256-frame 1080p video batch rendered on the device,
  split into contiguous frame blocks over the ranks (video.frame_block), each
  block filled in batched launches with no data-path collective ("weak" in
  the per-rank sense, the 256 frames are fixed: the same workload at every
  N).  Reported as ``c5`` on every line; it is ``value`` when N > 1.

Inputs are resident in HBM before the timed region (``value``); ``e2e``
repeats the metric through the public API with host buffers and the copies
inside the timed region.

Multi-GPU: ``--gpus N`` spawns N processes itself (one per GPU, NCCL
process group) unless it is already running under torchrun (WORLD_SIZE set).
Step times are CUDA-event times, max over ranks.

``--impl reference`` times the reference algorithm's CPU implementation (the
numpy port in oracle/, since the Python reference cannot travel to the GPU
box) on the same workload, over a process pool on all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpixels inpainted/s and ms per 1080p frame; fill-kernel HBM GB/s vs peak"
DTYPE = "f32 colour / f64 decisions"
C5_FRAMES = 256


def _ncu_traffic():
    """DRAM bytes of one fill launch: from the committed ncu --set full capture
    named in the returned source (ncu cannot run inside a timed bench)."""
    for name in ("round2_ncu_summary.json", "round1_ncu_summary.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                d = json.load(f)
            return float(d["fill_dram_bytes_per_launch"]), f"profiles/{name} ({d.get('head', '?')})"
        except Exception:
            continue
    return None, None


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

    def __init__(self, index=0, period_s=0.0005):
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
            # NVML's first query is slow: start timing once the poller runs
            t_end = time.time() + 1.0
            while not self.samples and time.time() < t_end:
                time.sleep(0.0002)
            self.samples.clear()
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
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, local


def b_frame(H, W, D, C=3):
    """Algorithmic bytes of one frame: fp32 image in + out,
    labels, g (2 x fp64) over D."""
    return H * W * (C * 4 + C * 4 + 1) + 16 * D


# ------------------------------------------------------------ CPU baselines

_POOL_SCENE = {}


def _pool_init(workload, counter, frames):
    from paper_1611_05319_b200 import scenes

    with counter.get_lock():
        k = counter.value
        counter.value += 1
    if workload == "C5":
        sc = scenes.config("C5", frame=frames[k % len(frames)])
    else:
        sc = scenes.config(workload)
    _POOL_SCENE["sc"] = sc


def _pool_task(_):
    from oracle import guidefill_oracle as orc

    sc = _POOL_SCENE["sc"]
    p = orc.Params(**sc.params)
    t0 = time.perf_counter()
    field = orc.guide_field([orc.polyline(s["points"], s["kind"]) for s in sc.splines],
                            [s["direction"] for s in sc.splines], sc.labels)
    orc.fill(sc.image, sc.labels, field, p, tracked=True)
    return sc.n_inpaint, time.perf_counter() - t0


def pool_baseline(workload, min_s=8.0, frames=None):
    """The reference algorithm (numpy port) over a process pool on every host
    core: one frame per task, guide field + full tracked fill, as BASELINE.md
    section 3 prescribes for the video batch.  Returns the Mpx/s of the timed
    rounds (scene generation is in the pool initialiser, not timed)."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    # spawned workers (the parent may hold a CUDA context and helper threads);
    # numpy stays single-threaded in each
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    ctx = mp.get_context("spawn")
    counter = ctx.Value("i", 0)
    frames = list(frames or range(cores))
    with ctx.Pool(cores, initializer=_pool_init, initargs=(workload, counter, frames)) as pool:
        pool.map(_pool_task, range(cores), chunksize=1)  # warm-up: one frame per worker
        t0 = time.perf_counter()
        done, px, rounds = [], 0, 0
        while True:
            out = pool.map(_pool_task, range(cores), chunksize=1)
            rounds += 1
            px += sum(d for d, _ in out)
            done.extend(t for _, t in out)
            if time.perf_counter() - t0 >= min_s:
                break
        wall = time.perf_counter() - t0
    return {"value": px / wall / 1e6, "unit": "Mpx/s", "cores": cores, "kind": "port",
            "sample": f"{rounds} rounds x {cores} {workload} frames (guide field + tracked fill, "
                      f"one frame per process, numpy restatement of the reference), {wall:.1f} s; "
                      f"single-core latency {statistics.median(done) * 1e3:.0f} ms/frame",
            "ms_per_frame_1core": statistics.median(done) * 1e3}


def run_reference(args):
    """Reference arm: the reference algorithm (numpy port) on the host cores,
    on this arm's workload: C2 frames at N = 1, C5 video frames at N > 1."""
    ws, rank, _ = dist_env()
    ws = max(ws, args.gpus)
    if rank != 0:
        return
    workload = "C2" if ws == 1 else "C5"
    # --steps K is honoured as "at least K frames per core" within the time bound
    cpu = pool_baseline(workload, min_s=min(60.0, max(8.0, 0.5 * args.steps)),
                        frames=list(range(C5_FRAMES)) if workload == "C5" else None)
    from paper_1611_05319_b200 import scenes

    sc = scenes.config(workload)
    value = cpu["value"]
    line = {
        "metric": METRIC, "value": value, "unit": "Mpx/s", "impl": "reference",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sc.n_inpaint / (value * 1e6) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": (f"C2 1920x1080 disocclusion frames, |D|={sc.n_inpaint}, r=3, "
                                f"mu=50, tracked, one frame per host process"
                                if workload == "C2" else
                                f"C5 1080p video frames (of {C5_FRAMES}), r=3, mu=50, tracked, "
                                f"one frame per host process"),
                   "global_batch": 1 if workload == "C2" else C5_FRAMES},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "Mpx/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU arm

def _flusher(dev):
    import torch

    flush_w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_r = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    sink = torch.empty(1, dtype=torch.float32, device=dev)

    def flush_l2():
        # evict L2 (126 MB): write 256 MB, then read another 256 MB so the
        # write-backs of the flush land outside the timed region
        flush_w.zero_()
        torch.sum(flush_r, dim=0, keepdim=True, out=sink)
    return flush_l2


def _timed(fn, steps, flush, clk_index):
    """CUDA-event times (ms) of ``steps`` calls of fn on the current stream."""
    import torch

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    torch.cuda.synchronize()
    with ClockSampler(clk_index) as clk:
        for k in range(steps):
            flush()
            starts[k].record()
            fn()
            ends[k].record()
        torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)], clk.summary()


def _spl_objs(raw):
    from paper_1611_05319_b200 import Spline

    return [Spline(id=x["id"], source="user", direction=x["direction"], points=x["points"],
                   kind=x["kind"]) for x in raw]


def bench_c2(args, dev, local):
    """C2 single frame: CUDA-graph replays of one gf_fill_splines call."""
    import numpy as np
    import torch

    from paper_1611_05319_b200 import FillParams, scenes
    from paper_1611_05319_b200 import _native as N
    from paper_1611_05319_b200._device import FillGraph, SegmentSet, fill_device

    sc = scenes.config(args.config)
    params = FillParams(**sc.params)
    H, W = sc.labels.shape
    D = sc.n_inpaint
    img = torch.from_numpy(sc.image[None].astype(np.float32)).to(dev).contiguous()
    lab = torch.from_numpy(sc.labels[None]).to(dev).contiguous()
    segs = SegmentSet(_spl_objs(sc.splines), dev)
    flush = _flusher(dev)
    ws_buf = None

    def step(trace_cap=0):
        nonlocal ws_buf
        res = fill_device(img, lab, None, params, tracked=not args.untracked, rows_cap=4096,
                          workspace=ws_buf, splines=segs, trace_cap=trace_cap)
        ws_buf = res["workspace"]
        return res

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        step()
    torch.cuda.synchronize()
    eager_ms = (time.perf_counter() - t0) / 20 * 1e3
    graph = FillGraph(img, lab, None, params, tracked=not args.untracked, rows_cap=4096,
                      splines=segs)
    for _ in range(max(3, args.warmup)):
        res = graph.replay()
    torch.cuda.synchronize()
    stats = res["stats"].cpu().numpy()
    assert int(stats[:, N.STAT_FILLED].sum()) == D, "fill incomplete"
    n_shells = int(stats[:, N.STAT_ITERATIONS].max())
    # per-shell phase trace of one (untimed) step
    res = step(trace_cap=256)
    torch.cuda.synchronize()
    tr = res["trace"].cpu().numpy()
    tl = tr[-1].astype(np.uint64)
    t_start = [int(~np.uint64(tl[2 * i])) for i in range(2)]
    t_end = [int(tl[2 * i + 1]) for i in range(2)]
    timeline = {name: {"start_us": (t_start[i] - t_start[0]) / 1e3,
                       "end_us": (t_end[i] - t_start[0]) / 1e3}
                for i, name in enumerate(["prep", "shells"])}
    shell_trace = []
    for r in tr[:n_shells]:
        row = {"items": int(r[5]), "fill_us": (r[1] - r[0]) / 1e3, "sync_us": (r[2] - r[1]) / 1e3}
        if args.untracked:
            row.update(rescan_us=(r[3] - r[2]) / 1e3, sync2_us=(r[4] - r[3]) / 1e3)
        shell_trace.append(row)
    step_ms, clocks = _timed(graph.replay, args.steps, flush, local)
    t = sum(step_ms) / len(step_ms)
    return dict(scene=sc, params=params, D=D, H=H, W=W, t_ms=t, step_ms=step_ms, clocks=clocks,
                shells=n_shells, timeline=timeline, shell_trace=shell_trace, eager_ms=eager_ms,
                launches=graph.launches_per_replay * args.steps)


def bench_c5(args, dev, ws, rank, local):
    """This rank's block of the C5 video batch, device-rendered, filled in
    batched chunks captured as one CUDA graph; one step = the whole block."""
    import torch

    from paper_1611_05319_b200 import FillParams, scenes
    from paper_1611_05319_b200 import _native as N
    from paper_1611_05319_b200._device import BatchGraph
    from paper_1611_05319_b200.video import frame_block

    blk = frame_block(args.c5_frames, ws, rank)
    t0 = time.perf_counter()
    images, labels, spl_raw = scenes.video_batch_device(list(blk), dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    sc0 = scenes.config("C5", frame=0)
    params = FillParams(**sc0.params)
    H, W = labels.shape[1:]
    D = int((labels == 255).sum().item())
    splines = [_spl_objs(s) for s in spl_raw]
    graph = BatchGraph(images, labels, splines, params, chunk=args.chunk,
                       tracked=not args.untracked, streams=args.streams)
    for _ in range(max(3, args.warmup)):
        graph.replay()
    torch.cuda.synchronize()
    st = graph.stats()
    assert int(st[:, N.STAT_FILLED].sum()) == D, "C5 fill incomplete"
    assert not st[:, N.STAT_UNFILLABLE].any()
    flush = _flusher(dev)
    step_ms, clocks = _timed(graph.replay, args.steps, flush, local)
    t = sum(step_ms) / len(step_ms)
    return dict(frames=len(blk), D=D, H=H, W=W, t_ms=t, step_ms=step_ms, clocks=clocks,
                gen_s=gen_s, launches=graph.launches_per_replay * args.steps,
                shells_max=int(st[:, N.STAT_ITERATIONS].max()), params=params,
                images=images, labels=labels, splines=splines, blk=blk)


def e2e_c2(c2, steps):
    """C2 end to end through tracker.run_tracked with host buffers."""
    import numpy as np
    import torch

    from paper_1611_05319_b200 import build_guide_field, tracker

    sc, params = c2["scene"], c2["params"]
    splines = _spl_objs(sc.splines)
    labels_h, image_h = sc.labels, sc.image
    holder = {}

    def timed(fn, n):
        # every call returns a host result (synchronous); the median of the
        # per-call wall times -- one slow call (a host page fault, a PCIe
        # hiccup) does not move it -- and the mean next to it
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(n):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        holder.setdefault("means", []).append(sum(ts) / n)
        return sorted(ts)[n // 2]

    ne = max(3, min(steps, 20))

    def fused():
        holder["u"], _ = tracker.run_tracked(image_h, labels_h, splines, params)

    def dropin():
        fld = build_guide_field(splines, labels_h)
        holder["u2"], _ = tracker.run_tracked(image_h, labels_h, fld, params)
        holder["fld"] = fld

    image_p = torch.from_numpy(image_h).pin_memory()
    labels_p = torch.from_numpy(labels_h).pin_memory()

    def pinned():
        holder["up"], _ = tracker.run_tracked(image_p, labels_p, splines, params)

    tp = timed(pinned, ne)
    te = timed(fused, ne)
    td = timed(dropin, ne)
    u, fld = holder["u"], holder["fld"]
    assert np.array_equal(holder["up"].numpy(), u), "pinned path differs from the numpy path"
    delta_px = int((u.view(np.uint64) != np.ascontiguousarray(image_h).view(np.uint64))
                   .any(axis=2).sum())
    D = c2["D"]
    return {"value": D / tp / 1e6, "unit": "Mpx/s", "ms_per_frame": tp * 1e3,
            "ms_per_frame_mean": holder["means"][0] * 1e3,
            "timing": f"median of {ne} synchronous calls (wall clock), mean alongside",
            "h2d_bytes_per_step": int(image_h.nbytes + labels_h.nbytes),
            # the result buffer is seeded with the input by D2H DMA as the
            # upload lands, then the changed pixels are written after the fill
            "d2h_bytes_per_step": int(u.nbytes + delta_px * u.shape[2] * u.itemsize),
            "d2h_delta_px": delta_px,
            "path": "tracker.run_tracked(image, labels, splines, params) on pinned host tensors "
                    "(f64 image in, f64 image out, copies in the timed region); the result buffer "
                    "is seeded with the input by D2H DMA while the upload runs "
                    "(gf_upload_mirrored), then gf_output_delta writes the changed pixels",
            "numpy_ms_per_frame": te * 1e3,
            "numpy_path": "the same call on pageable numpy f64 arrays (the reference's types)",
            "dropin_two_call_ms": td * 1e3,
            "dropin_two_call_bytes": int(image_h.nbytes + 2 * labels_h.nbytes + 2 * fld.nbytes
                                         + u.nbytes)}


def e2e_c5(c5, ring=16):
    """This rank's C5 block end to end from pinned host memory: the frames
    stream through video.fill_video_host (uploads, fills and downloads of
    consecutive frames overlap on three streams); host f64 frames come from a
    ring of ``ring`` distinct frames of the block, each with its own mask and
    splines.  Timed with CUDA events on the caller's stream."""
    import torch

    from paper_1611_05319_b200 import video

    n = c5["frames"]
    ring = min(ring, n)
    h_img = [c5["images"][i].to(torch.float64).cpu().pin_memory() for i in range(ring)]
    h_lab = [c5["labels"][i].cpu().pin_memory() for i in range(ring)]
    d_ring = [int((c5["labels"][i] == 255).sum().item()) for i in range(ring)]
    seq = [i % ring for i in range(n)]
    filled = []

    def consume(f, u, rep):
        filled.append(rep.filled)

    imgs = [h_img[i] for i in seq]
    labs = [h_lab[i] for i in seq]
    spls = [c5["splines"][i] for i in seq]
    video.fill_video_host(imgs[:ring], labs[:ring], spls[:ring], c5["params"], on_frame=consume)
    torch.cuda.synchronize()
    filled.clear()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    video.fill_video_host(imgs, labs, spls, c5["params"], on_frame=consume)
    e1.record()
    torch.cuda.synchronize()
    t_ms = e0.elapsed_time(e1)
    D = sum(d_ring[i] for i in seq)
    assert sum(filled) == D
    fb = h_img[0].numel() * 8
    return {"t_ms": t_ms, "D": D, "frames": n,
            "h2d_bytes_per_step": int(n * (fb + h_lab[0].numel())),
            "d2h_bytes_per_step": int(n * fb)}


def bench_deadlock(dev):
    """SURVEY.md section 7 hard part 2: the 256x256 half-plane at 25 degrees,
    smart order, mu 50 -- 22,058 shells, 16,636 of them deadlock-guarded
    (tests/cases.deadlock_scenes, parity in tests/test_gpu_deadlock.py)."""
    import numpy as np
    import torch

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import cases

    from paper_1611_05319_b200 import FillParams
    from paper_1611_05319_b200 import _native as N
    from paper_1611_05319_b200._device import fill_device

    out = {}
    for th in (25.0, 10.0):
        case = cases.deadlock_scenes(thetas=(th,), mus=(50.0,))[0]
        img = torch.from_numpy(case["image"][None].astype(np.float32)).to(dev)
        lab = torch.from_numpy(case["labels"][None]).to(dev)
        g = torch.from_numpy(case["guide"][None]).to(dev)
        p = FillParams(**case["params"])
        res = fill_device(img, lab, g, p, rows_cap=1 << 16)
        ws = res["workspace"]
        # median of 3 timed fills: this runs right after the CPU pool
        # baseline, and the first fill after seconds of GPU idle can run
        # while the clocks ramp back up (measured 19.6 vs 11.6 us per shell)
        runs = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            res = fill_device(img, lab, g, p, rows_cap=1 << 16, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            runs.append(e0.elapsed_time(e1))
        st = res["stats"][0].cpu().numpy()
        ms = sorted(runs)[1]
        out[case["name"]] = {"ms": ms, "ms_runs": runs, "shells": int(st[N.STAT_ITERATIONS]),
                             "guarded_shells": int(st[N.STAT_DEADLOCK]),
                             "us_per_shell": ms * 1e3 / int(st[N.STAT_ITERATIONS])}
    a, b = out["halfplane_25deg_mu50"], out["halfplane_10deg_mu50"]
    # per guarded shell: the 10 degree chain is 97% unguarded shells of the
    # same kind, so its us/shell prices the unguarded part of the 25 degree one
    a["us_per_guarded_shell_est"] = ((a["ms"] * 1e3 - (a["shells"] - a["guarded_shells"])
                                      * b["us_per_shell"]) / a["guarded_shells"])
    return out


def bench_coherence(dev, reps=7):
    """the coherence-transport preset (FillParams.coherence_transport:
    g from the masked structure tensor every shell) on the C2 frame -- the whole
    fill in one persistent kernel (coherence.run_coherence_fill); device-resident
    f64 frame, and through the public API from host numpy arrays."""
    import numpy as np
    import torch

    from paper_1611_05319_b200 import FillParams, engine, scenes
    from paper_1611_05319_b200.coherence import run_coherence_fill

    sc = scenes.config("C2")
    p = FillParams.coherence_transport()
    img = torch.from_numpy(np.ascontiguousarray(sc.image, dtype=np.float64)).to(dev)
    lab = torch.from_numpy(sc.labels).to(dev)
    for _ in range(2):
        run_coherence_fill(img.clone(), lab, p, tracked=True)
    ts = []
    rep = None
    for _ in range(reps):
        u = img.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, rep, _, _ = run_coherence_fill(u, lab, p, tracked=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    engine.coherence_transport_mode(sc.image, sc.labels)  # warm-up
    t0 = time.perf_counter()
    engine.coherence_transport_mode(sc.image, sc.labels)
    api_ms = (time.perf_counter() - t0) * 1e3
    return {"ms_per_frame": min(ts), "ms_median": sorted(ts)[len(ts) // 2], "ms_all": ts,
            "shells": rep["iterations"], "filled": rep["filled"],
            "mpx_s": rep["filled"] / (min(ts) * 1e3),
            "host_api_ms": api_ms,
            "host_api_path": "engine.coherence_transport_mode(numpy f64 image, labels)",
            "path": "coherence.run_coherence_fill: one cooperative launch of k_ct_loop "
                    "(gf_coherence_fill) for all shells, f64 frame resident, one host sync",
            "workload": "C2 1920x1080, 77,440 Inpaint px, r=5 axis ball, onion, "
                        "sigma 2, rho 4, lambda 1e-5"}


def bench_detect():
    """Automatic spline detection (guide.detect_splines) on the C2 and C4
    frames through the public API (host f64 image in, Spline list out)."""
    from paper_1611_05319_b200 import guide, scenes

    out = {}
    for name in ("C2", "C4"):
        sc = scenes.config(name)
        guide.detect_splines(sc.image, sc.labels)  # warm-up
        t0 = time.perf_counter()
        spl = guide.detect_splines(sc.image, sc.labels)
        out[name] = {"ms": (time.perf_counter() - t0) * 1e3, "splines": len(spl),
                     "path": "guide.detect_splines: gf_detect_edges (ring, Canny, seed strengths), "
                             "host clustering, gf_structure_eigen, gf_trace_rays"}
    return out


def rank_main(args):
    import torch
    import torch.distributed as dist

    from paper_1611_05319_b200 import _native as N

    ws, rank, local = dist_env()
    # GF_BENCH_ONE_DEVICE=1: every rank on device 0 with gloo -- a functional
    # check of the multi-rank path on a one-GPU box (times are not measurements:
    # the ranks share the GPU)
    one_dev = os.environ.get("GF_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    launches0 = N.launch_count()

    from paper_1611_05319_b200.video import reduce_over_ranks

    def job_max(x):
        return reduce_over_ranks(maxes=[x], device=dev)[1][0]

    def job_sum(x):
        return reduce_over_ranks(sums=[x], device=dev)[0][0]

    c2 = bench_c2(args, dev, local) if ws == 1 else None
    if ws > 1:
        dist.barrier()
    c5 = bench_c5(args, dev, ws, rank, local) if not args.no_c5 else None
    peak, peak_kind = _peaks()
    c5_line = None
    if c5 is not None:
        t_job = job_max(c5["t_ms"])
        D_job = job_sum(c5["D"])
        bytes_rank = c5["frames"] * b_frame(c5["H"], c5["W"], 0) + 16 * c5["D"]
        bytes_job = job_sum(bytes_rank)
        ach = bytes_rank / (c5["t_ms"] * 1e-3) / 1e9
        c5_line = {
            "value": D_job / (t_job * 1e-3) / 1e6, "unit": "Mpx/s",
            "frames_total": args.c5_frames, "frames_per_gpu": c5["frames"],
            "ms_per_step": t_job, "ms_per_frame_per_gpu": c5["t_ms"] / c5["frames"],
            "inpaint_px_total": int(D_job), "shells_max": c5["shells_max"],
            "chunk": args.chunk, "ms_step_min": min(c5["step_ms"]),
            "ms_step_max": max(c5["step_ms"]),
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": ach / peak,
                         "algorithmic_bytes_per_gpu": bytes_rank,
                         "algorithmic_bytes_job": bytes_job},
            "workload": f"C5: {args.c5_frames} device-rendered 1080p frames (seeds 1611 + 7919 f, "
                        f"objects drifting 3 px/frame), contiguous blocks per GPU, batched "
                        f"gf_fill_splines in chunks of {args.chunk} frames, one CUDA graph",
            "render_s": c5["gen_s"],
            "clocks": c5["clocks"],
        }
        if not args.no_e2e:
            e = e2e_c5(c5)
            te = job_max(e["t_ms"])
            De = job_sum(e["D"])
            c5_line["e2e"] = {
                "value": De / (te * 1e-3) / 1e6, "unit": "Mpx/s", "ms_per_step": te,
                "ms_per_frame_per_gpu": te / e["frames"],
                "h2d_bytes_per_step": int(job_sum(e["h2d_bytes_per_step"])),
                "d2h_bytes_per_step": int(job_sum(e["d2h_bytes_per_step"])),
                "path": "video.fill_video_host per GPU over its block (pinned f64 host frames "
                        "from a ring of 16 distinct frames of the block, own masks and splines; "
                        "H2D, fill and D2H of consecutive frames overlap on three streams)"}
        del c5["images"], c5["labels"]
    launches = N.launch_count() - launches0
    if ws > 1:
        dist.barrier()
    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    traffic, traffic_src = _ncu_traffic()
    if ws == 1:
        sc = c2["scene"]
        D = c2["D"]
        bf = b_frame(c2["H"], c2["W"], D)
        ach = bf / (c2["t_ms"] * 1e-3) / 1e9
        e2e = None if args.no_e2e else e2e_c2(c2, args.steps)
        if e2e is not None and c5_line is not None and "e2e" in c5_line:
            e2e["video_pipelined_mpx_s"] = c5_line["e2e"]["value"]
            e2e["video_pipelined_ms_per_frame"] = c5_line["e2e"]["ms_per_frame_per_gpu"]
        cpu = None if args.no_cpu else pool_baseline("C2")
        deadlock = None if args.no_extras else bench_deadlock(dev)
        detect = None if args.no_extras else bench_detect()
        coherence = None if args.no_extras else bench_coherence(dev)
        line = {
            "metric": METRIC, "value": D / (c2["t_ms"] * 1e-3) / 1e6, "unit": "Mpx/s",
            "n_gpus": 1, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": c2["t_ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": {
                "workload": f"{sc.name} 1920x1080 disocclusion frame: guide-field raster + "
                            f"{'untracked' if args.untracked else 'tracked'} shell fill, "
                            f"fp32 RGB in/out, fp64 decisions",
                "global_batch": 1, "inpaint_px": D, "shells": c2["shells"],
                "r": sc.params["r"], "mu": sc.params["mu"], "ms_per_frame": c2["t_ms"],
                "ms_step_min": min(c2["step_ms"]), "ms_step_max": max(c2["step_ms"]),
                "timeline": c2["timeline"], "shell_trace": c2["shell_trace"],
                "l2": "flushed between steps (256 MB write + 256 MB read, untimed)",
                "launch": "CUDA graph replay of memset + k_prep + k_shells",
                "eager_host_ms_per_call": c2["eager_ms"], "parallelism": "single frame",
            },
            "roofline": {"bound": "hbm", "kernel": "gf_fill_splines (k_prep + k_shells)",
                         "achieved": ach, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": ach / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_bytes": bf},
            "e2e": e2e,
            "c5": c5_line,
            "deadlock_regime": deadlock,
            "spline_detection": detect,
            "coherence_transport": coherence,
            "gpu_launches": c2["launches"],
            "gpu_launches_note": "library kernels (gf_launch_count) in the C2 timed replays; "
                                 "the whole run launched "
                                 f"{launches} incl. C5 ({c5['launches'] if c5 else 0} timed)",
            "clocks": c2["clocks"],
            "cpu_baseline": cpu,
        }
    else:
        line = {
            "metric": METRIC, "value": c5_line["value"], "unit": "Mpx/s", "n_gpus": ws,
            "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": c5_line["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": {"workload": c5_line["workload"], "global_batch": args.c5_frames,
                       "frames_per_gpu": c5_line["frames_per_gpu"],
                       "parallelism": f"frame-parallel x{ws}, no data-path collective",
                       "l2": "flushed between steps; each step's inputs exceed L2"},
            "roofline": dict(c5_line["roofline"], traffic=None,
                             traffic_source="per-frame ncu capture: see the N=1 line"),
            "e2e": c5_line.get("e2e"),
            "c5": c5_line,
            "gpu_launches": c5["launches"],
            "clocks": c5_line["clocks"],
            "cpu_baseline": None,
        }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _spawned(local, world, port, argv):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(local),
                      LOCAL_RANK=str(local), WORLD_SIZE=str(world), LOCAL_WORLD_SIZE=str(world))
    rank_main(parse(argv))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--untracked", action="store_true")
    ap.add_argument("--c5-frames", type=int, default=C5_FRAMES)
    ap.add_argument("--chunk", type=int, default=64, help="frames per batched launch (C5)")
    ap.add_argument("--streams", type=int, default=1,
                    help="streams the C5 chunks alternate over (overlap of prep and shells)")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the deadlock-regime and spline-detection timings")
    return ap.parse_args(argv)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not under torchrun: one process per GPU, spawned here
        import torch.multiprocessing as mp

        mp.spawn(_spawned, args=(args.gpus, _free_port(), sys.argv[1:]), nprocs=args.gpus,
                 join=True)
        return
    rank_main(args)


if __name__ == "__main__":
    main()
