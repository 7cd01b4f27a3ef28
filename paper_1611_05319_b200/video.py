"""Frame-parallel video fill (BASELINE.json config C5).

Frames of a video are independent fills, so a batch is
partitioned into contiguous frame blocks, one block per GPU / rank, with no
data-path collective: every rank fills its block with one batched
gf_fill_splines launch.  Collectives are used only for bookkeeping (the
max-over-ranks timing, optional result gathers), never inside the fill.
"""

from __future__ import annotations

import numpy as np


def frame_block(n_frames: int, world: int, rank: int) -> range:
    """Contiguous block of frames owned by ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def reduce_over_ranks(sums=(), maxes=(), device="cpu"):
    """Job-wide totals of per-rank numbers for a frame-parallel run: ``sums``
    (inpainted pixels, bytes) added over the ranks, ``maxes`` (step times)
    maximised -- the job takes as long as its slowest rank.  Collectives run
    on the process group torch.distributed was initialised with (NCCL on the
    GPUs, gloo in the CPU tests); without one the inputs come back as they are.
    These are bookkeeping collectives, never on the fill's data path."""
    import torch
    import torch.distributed as dist

    sums, maxes = [float(x) for x in sums], [float(x) for x in maxes]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return sums, maxes
    out = []
    for vals, op in ((sums, dist.ReduceOp.SUM), (maxes, dist.ReduceOp.MAX)):
        if not vals:
            out.append([])
            continue
        # gloo reduces host tensors; NCCL device ones
        dev = "cpu" if dist.get_backend() == "gloo" else device
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=op)
        out.append(t.cpu().tolist())
    return out[0], out[1]


def frame_checksum(u: np.ndarray) -> float:
    """Order-independent digest used to compare per-frame results across ranks."""
    return float(np.asarray(u, dtype=np.float64).sum())


def fill_video(images, labels, splines, params, tracked=True, device=None, workspace=None):
    """Fill a (N, H, W, C) batch of frames that share one spline set.

    images: float32/float64 CUDA tensor (N, H, W, C); labels: uint8 CUDA
    tensor (N, H, W); splines: a ``_device.SegmentSet`` or None (g = 0).
    Returns the ``fill_device`` result dict (out, stats, rows, ...).
    """
    from ._device import fill_device

    return fill_device(images, labels, None, params, tracked=tracked, splines=splines,
                       workspace=workspace)


def _frame_hw(x):
    return tuple(int(d) for d in x.shape[:2])


def _check_video_masks(images, labels):
    """Labels of a video: one (H, W) mask shared by every frame, a sequence of
    per-frame masks, or an (N, H, W) stack of them (returned as a list).  Every
    mask must match its frame's (H, W) -- a mismatch would make the kernels
    read past the device labels -- and the reference's "differ" ValueError is
    raised otherwise (engine.py:398-401)."""
    n = len(images)
    if not isinstance(labels, (list, tuple)):
        nd = len(labels.shape)
        if nd == 3:
            if int(labels.shape[0]) != n:
                raise ValueError(f"{int(labels.shape[0])} label masks for {n} frames")
            labels = [labels[f] for f in range(n)]
        elif nd != 2:
            raise ValueError("labels must be one (H, W) mask, a sequence of them or an "
                             "(N, H, W) stack")
    if isinstance(labels, (list, tuple)):
        if len(labels) != n:
            raise ValueError(f"{len(labels)} label masks for {n} frames")
        for f in range(n):
            if len(labels[f].shape) != 2 or _frame_hw(labels[f]) != _frame_hw(images[f]):
                raise ValueError(f"frame {f}: image and label shapes differ")
    else:
        for f in range(n):
            if _frame_hw(labels) != _frame_hw(images[f]):
                raise ValueError(f"frame {f}: image and label shapes differ")
    return labels


_streams = {}


def _pipeline_streams(dev):
    import threading

    import torch

    key = (str(dev), threading.get_ident())
    got = _streams.get(key)
    if got is None:
        got = tuple(torch.cuda.Stream(device=dev) for _ in range(3))
        _streams[key] = got
    return got


def fill_video_host(images, labels, splines, params, tracked=True, depth=3, on_frame=None):
    """Fill a sequence of HOST frames with transfers and fills pipelined.

    images: sequence of (H, W, C) frames, float64 numpy arrays or pinned CPU
    tensors (what a decoder writing into page-locked buffers hands over);
    labels: one (H, W) uint8 mask shared by all frames, a sequence of
    per-frame masks, or an (N, H, W) stack of them (each checked against its
    frame's shape); splines: a Spline list shared by all frames (rastered inside each
    fill), a sequence of per-frame Spline lists, or None for g = 0.
    Returns [(u, FillReport)] in frame order, u of the input's kind (numpy
    float64 / pinned CPU tensor).

    Three streams: uploads, fills (one stream, so the cooperative shell
    kernels never run side by side) and downloads.  While frame n fills,
    frame n+1 uploads and frame n-1 downloads: the PCIe link carries both
    directions at once and the fill hides under the transfers.  ``depth``
    frames are in flight.  Per-frame results equal ``tracker.run_tracked``
    (tests/test_gpu_configs.py).

    With ``on_frame(f, u, report)`` each result is handed over in frame order
    as soon as it lands and is not retained (returns None): a streaming
    consumer keeps the pinned result buffers recycling instead of pinning
    new host memory for every frame.
    """
    import torch

    from . import _native as N
    from ._device import SegmentSet
    from .engine import _report_from, _run_fill

    dev = N.require_cuda()
    n = len(images)
    if n == 0:
        return []
    depth = max(1, int(depth))
    labels = _check_video_masks(images, labels)
    shared_lab = not isinstance(labels, (list, tuple))
    per_frame_spl = bool(splines) and isinstance(splines[0], (list, tuple))
    segs = SegmentSet.cached(list(splines), dev) if splines and not per_frame_spl else None
    # the same three streams on every call: torch's caching allocator keeps
    # freed blocks per stream, so fresh streams would cudaMalloc every frame
    # buffer anew (and stall on cudaFree when the cache is trimmed)
    s_up, s_fill, s_down = _pipeline_streams(dev)
    caller = torch.cuda.current_stream()
    for s in (s_up, s_fill, s_down):
        s.wait_stream(caller)  # labels / segments the caller's stream produced
    stage = [None] * depth
    lab_stage = [None] * depth
    rep_bufs = [None] * depth
    d_lab_shared = None
    if shared_lab:
        lab0 = np.asarray(labels)
        d_lab_shared = torch.from_numpy(np.ascontiguousarray(lab0, dtype=np.uint8)).to(dev)
        d_lab_shared = d_lab_shared.reshape(1, *lab0.shape)
        for s in (s_up, s_fill, s_down):
            s.wait_stream(caller)
    pending = [None] * depth
    results = [None] * n

    def finish(slot):
        f, ev, u_host, u_ret, st_h, rw_h, _keep = pending[slot]
        ev.synchronize()
        H, W = u_host.shape[:2]
        stats = st_h.numpy()
        rows = rw_h.numpy()
        if stats[N.STAT_BAD_LABELS]:
            # k_prep saw a label outside {0, 128, 255}: the reference's ValueError
            from . import grid

            lab_f = labels if shared_lab else labels[f]
            grid.validate_labels(np.asarray(lab_f.numpy() if isinstance(lab_f, torch.Tensor)
                                            else lab_f))
            raise ValueError("label mask holds values outside {0, 128, 255}")
        if stats[N.STAT_UNFILLABLE] or int(stats[N.STAT_ITERATIONS]) + 1 > rows.shape[0]:
            # rare: stranded pixels (the device EDT paint) or a report longer
            # than the pipeline's row buffer -- the single-frame path handles both
            lab_f = labels if shared_lab else labels[f]
            spl_f = splines[f] if per_frame_spl else splines
            u, rep, _ = _run_fill(images[f], lab_f, None, params, tracked, splines=spl_f)
        else:
            u, rep = u_ret, _report_from(stats, rows, tracked, H, W)
        pending[slot] = None
        if on_frame is not None:
            on_frame(f, u, rep)
        else:
            results[f] = (u, rep)

    try:
        _pipeline(n, depth, pending, finish, images, labels, splines, params, tracked, dev,
                  shared_lab, d_lab_shared, per_frame_spl, segs, stage, lab_stage, rep_bufs,
                  s_up, s_fill, s_down)
    except BaseException:
        # in-flight copies still target pooled host buffers: drain before unwinding
        for s_ in (s_up, s_fill, s_down):
            s_.synchronize()
        raise
    caller.wait_stream(s_down)
    return None if on_frame is not None else results


def _pipeline(n, depth, pending, finish, images, labels, splines, params, tracked, dev,
              shared_lab, d_lab_shared, per_frame_spl, segs, stage, lab_stage, rep_bufs,
              s_up, s_fill, s_down):
    """The frame loop of fill_video_host (enqueue frame f, retire frame f - depth)."""
    import torch

    from . import _native as N
    from . import _staging
    from ._device import SegmentSet, fill_device

    ws = None
    for f in range(n):
        slot = f % depth
        if pending[slot] is not None:
            finish(slot)
        src = images[f]
        as_tensor = isinstance(src, torch.Tensor)
        if as_tensor and src.is_pinned() and src.dtype == torch.float64 and src.is_contiguous():
            h_img = src
        else:
            a = np.ascontiguousarray(src.numpy() if as_tensor else src, dtype=np.float64)
            if stage[slot] is None or stage[slot].numel() < a.size:
                stage[slot] = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
            h_img = stage[slot][:a.size].view(a.shape)
            np.copyto(h_img.numpy(), a)  # this slot's previous upload has finished
        H, W, C = h_img.shape
        with torch.cuda.stream(s_fill):
            d_img = torch.empty((1, H, W, C), dtype=torch.float64, device=dev)
            d_lab = d_lab_shared if shared_lab else torch.empty((1, H, W), dtype=torch.uint8,
                                                                device=dev)
        with torch.cuda.stream(s_up):
            d_img.view(H, W, C).copy_(h_img, non_blocking=True)
            h_lab = None
            if not shared_lab:
                lf = labels[f]
                if isinstance(lf, torch.Tensor) and lf.is_pinned() and lf.dtype == torch.uint8:
                    h_lab = lf.contiguous()
                else:
                    la = np.ascontiguousarray(lf.numpy() if isinstance(lf, torch.Tensor) else lf,
                                              dtype=np.uint8)
                    if lab_stage[slot] is None or lab_stage[slot].numel() < la.size:
                        lab_stage[slot] = torch.empty(la.size, dtype=torch.uint8, pin_memory=True)
                    h_lab = lab_stage[slot][:la.size].view(la.shape)
                    np.copyto(h_lab.numpy(), la)  # this slot's previous upload has finished
                d_lab.view(H, W).copy_(h_lab, non_blocking=True)
            up = torch.cuda.Event()
            up.record()
        s_fill.wait_event(up)
        with torch.cuda.stream(s_fill):
            seg_f = segs
            if per_frame_spl:
                seg_f = SegmentSet.cached(list(splines[f]), dev) if len(splines[f]) else None
            res = fill_device(d_img, d_lab, None, params, tracked=tracked, rows_cap=4096,
                              workspace=ws, splines=seg_f)
            ws = res["workspace"]
            done = torch.cuda.Event()
            done.record()
        s_down.wait_event(done)
        with torch.cuda.stream(s_down):
            if as_tensor:
                u_host, _ = _staging._pool_out.take_tensor((H, W, C), torch.float64)
                u_ret = u_host
            else:
                u_ret, buf = _staging._pool_out.take((H, W, C), np.float64)
                u_host = buf[:u_ret.nbytes].view(torch.float64).view(H, W, C)
            u_host.copy_(res["out"][0], non_blocking=True)
            if rep_bufs[slot] is None:
                rep_bufs[slot] = (torch.empty(N.GF_STATS, dtype=torch.int32, pin_memory=True),
                                  torch.empty((4096, 2), dtype=torch.int32, pin_memory=True))
            st_h, rw_h = rep_bufs[slot]
            st_h.copy_(res["stats"][0], non_blocking=True)
            rw_h.copy_(res["rows"][0], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
        # device buffers stay referenced until the download event has passed
        pending[slot] = (f, ev, u_host, u_ret, st_h, rw_h, (d_img, d_lab, res, h_img, h_lab))
    for k in range(n, n + depth):
        if pending[k % depth] is not None:
            finish(k % depth)


def fill_video_multi(images, labels, splines, params, devices=None, tracked=True, depth=3,
                     on_frame=None):
    """Frame-parallel fill of a host video over several GPUs of one process.

    The frames are split into contiguous blocks (``frame_block``), one per
    device, and each block streams through ``fill_video_host`` on its own
    host thread with that device current: uploads, fills and downloads of
    different GPUs run concurrently (each GPU has its own PCIe link and
    copy engines) and no data crosses between devices.  Per-frame results
    are identical whatever the device count (each frame is one independent
    fill).

    images / labels / splines as for ``fill_video_host`` (labels: a shared
    mask, a per-frame sequence or an (N, H, W) stack).  devices: CUDA device
    indices or torch devices, default all visible GPUs.  Returns
    [(u, FillReport)] in frame order, or None with ``on_frame(f, u, report)``
    (called from the device threads, frames of one device in order).
    """
    import threading

    import torch

    from . import _native as N

    N.require_cuda()
    n = len(images)
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
    if not devices:
        raise ValueError("no devices to fill on")
    labels = _check_video_masks(images, labels)
    per_frame_spl = bool(splines) and isinstance(splines[0], (list, tuple))
    results = [None] * n
    errors = []

    def work(k, dev):
        blk = frame_block(n, len(devices), k)
        if len(blk) == 0:
            return
        idx = list(blk)
        lab = labels if not isinstance(labels, (list, tuple)) else [labels[f] for f in idx]
        spl = [splines[f] for f in idx] if per_frame_spl else splines
        cb = None
        if on_frame is not None:
            def cb(i, u, rep):
                on_frame(idx[i], u, rep)
        try:
            with torch.cuda.device(dev):
                out = fill_video_host([images[f] for f in idx], lab, spl, params,
                                      tracked=tracked, depth=depth, on_frame=cb)
                torch.cuda.current_stream().synchronize()
            if out is not None:
                for i, f in enumerate(idx):
                    results[f] = out[i]
        except BaseException as e:  # re-raised on the caller's thread
            errors.append(e)

    if len(devices) == 1:
        work(0, devices[0])
    else:
        threads = [threading.Thread(target=work, args=(k, d)) for k, d in enumerate(devices)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    if errors:
        raise errors[0]
    return None if on_frame is not None else results
