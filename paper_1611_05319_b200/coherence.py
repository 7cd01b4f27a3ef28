"""Coherence-transport fill (g_source = "modified_structure_tensor") on the GPU.

The reference resolves g per shell from the current image (engine._resolve_g,
engine.py:243-249 -> guide.coherence_directions, guide.py:330-355): every
shell's guidance reads the pixels the previous shell filled, so g cannot be
precomputed the way the guide field is.  This loop therefore runs shell by
shell from the host, with every per-pixel step on the device:

* g at the frontier: gf_coherence_directions (csrc/gf_coherence.cu, the masked
  structure tensor of guide._tensor_field as separable passes over the frame);
* weights, ghost gathers, masses and colours: gf_sample_points (the same ball
  evaluator the persistent shell kernel uses, engine.py:131-199);
* ready predicate, fill mask, scatter and relabel (engine.py:317-356):
  gf_commit_shell; the deadlock guard (one pixel) with torch device ops;
* tracked frontier update (tracker.py:59-79): gf_frontier_candidates marks the
  candidates and their active flag in one pass;
* unfillable fallback: gf_paint_unfillable.

The host only reads the frontier size and "anything filled?" per shell (the
loop's own control flow, engine.py:304-348).  Structure follows
engine._fill_loop (engine.py:286-376) step for step.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _native as N
from ._device import boundary_device, sample_points_device
from .grid import INPAINT, NEIGHBOR_OFFSETS, READABLE


def coherence_directions_device(u, lab, idx, sigma=2.0, rho=4.0, lam=1e-5, workspace=None,
                                points=None):
    """guide.coherence_directions (guide.py:330-355) at flat pixel indices ``idx``
    (int64 CUDA tensor): (n, 2) float64 CUDA tensor.  ``points`` (optional (n, 2)
    float64 CUDA tensor) receives the queries' (x, y)."""
    import torch

    lib = N.load()
    H, W, C = u.shape
    n = int(idx.numel())
    g = torch.empty((n, 2), dtype=torch.float64, device=u.device)
    need = lib.gf_coherence_workspace_bytes(H, W, C)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=u.device)
    N.check(lib.gf_coherence_directions(H, W, C, N.ptr(u), N.ptr(lab), n, N.ptr(idx),
                                        float(sigma), float(rho), float(lam), N.ptr(g),
                                        N.ptr(points), N.ptr(workspace), need, N.stream_ptr()))
    return g


def _active(lab, periodic_x):
    """grid.active_boundary_mask (grid.py:59-76) on the device, flattened."""
    return boundary_device(lab, periodic_x)[0].reshape(-1)


def _neighbor_mean(u, lab, p, H, W, periodic_x):
    """engine._neighbor_mean (engine.py:252-267): readable 8-neighbours, fixed order.

    The 3x3 block comes to the host and the mean is numpy's (sequential sum,
    then a true division: torch divides a CUDA tensor by a Python scalar as a
    multiplication by its reciprocal, one ulp off)."""
    import torch

    C = u.shape[2]
    j, i = divmod(p, W)
    rows = [jj for jj in (j - 1, j, j + 1) if 0 <= jj < H]
    cols = [(i + di) % W if periodic_x else i + di for di in (-1, 0, 1)]
    keep = [c for c in cols if 0 <= c < W]
    idx = torch.tensor([jj * W + c for jj in rows for c in keep], device=u.device)
    vals = u.reshape(-1, C)[idx].cpu().numpy()
    labs = lab.reshape(-1)[idx].cpu().numpy()
    pos = {int(q): k for k, q in enumerate(idx.tolist())}
    acc = np.zeros(C)
    n = 0
    for di, dj in NEIGHBOR_OFFSETS:
        ii, jj = i + di, j + dj
        if periodic_x:
            ii %= W
        if 0 <= ii < W and 0 <= jj < H and labs[pos[jj * W + ii]] == READABLE:
            acc += vals[pos[jj * W + ii]]
            n += 1
    if n == 0:
        return None
    return torch.from_numpy(acc / n).to(u.device)


_PINNED = {}


def _pinned_report(n):
    """A reusable pinned int32 host buffer per stream (page-locking per call
    costs more than the fill's last shells)."""
    import torch

    key = (torch.cuda.current_stream().cuda_stream, n)
    buf = _PINNED.get(key)
    if buf is None:
        buf = _PINNED[key] = torch.empty(n, dtype=torch.int32, pin_memory=True)
    return buf


_SCRATCH = {}


def _scratch(dev, H, W, C, cap):
    """Report rows, report and workspace of gf_coherence_fill, kept per (device,
    stream, geometry): the kernel initialises what it reads, and calls on one
    stream run in order, so they are reused as is."""
    import torch

    key = (str(dev), torch.cuda.current_stream(dev).cuda_stream, H, W, C)
    hit = _SCRATCH.pop(key, None)
    if hit is not None:
        _SCRATCH[key] = hit  # most recent last
    else:
        while len(_SCRATCH) >= 4:  # a few hundred MB each at 1080p: keep the last four
            _SCRATCH.pop(next(iter(_SCRATCH)))
        lib = N.load()
        ws_bytes = lib.gf_coherence_fill_workspace_bytes(H, W, C, cap)
        hit = _SCRATCH[key] = (torch.empty((cap + 1, 5), dtype=torch.int64, device=dev),
                               torch.empty(4, dtype=torch.int32, device=dev),
                               torch.empty(ws_bytes, dtype=torch.uint8, device=dev), ws_bytes)
    return hit


def run_coherence_fill(u, lab0, params, tracked=True, order_log=False):
    """engine._fill_loop (engine.py:286-376) with g from the masked structure tensor:
    the whole loop in one persistent kernel (gf_coherence_fill).

    ``u``: (H, W, C) float64 CUDA tensor (consumed: filled in place); ``lab0``:
    (H, W) uint8 CUDA tensor (not modified).  Returns (u, report fields dict,
    enter, fillshell) with the order maps as int32 CUDA tensors (enter None
    unless order_log).  A sigma window wider than the fused tile supports
    (sigma > 3.25) runs the shell-by-shell loop (``run_coherence_fill_shells``).
    """
    import torch

    from ._device import params_to_c

    H, W, C = u.shape
    dev = u.device
    lab = lab0.clone()
    lib = N.load()
    cap = H * W  # frontier capacity: >= the Inpaint count, no host count needed
    fillshell = torch.empty(H * W, dtype=torch.int32, device=dev)  # the kernel presets -1
    enter = torch.empty(H * W, dtype=torch.int32, device=dev) if order_log else None
    rows, report, ws, ws_bytes = _scratch(dev, H, W, C, cap)
    pc = params_to_c(params, tracked, N.GF_G_FIELD)
    t0 = time.perf_counter()
    rc = lib.gf_coherence_fill(H, W, C, N.ptr(u), N.ptr(lab), ctypes.byref(pc),
                               float(params.sigma), float(params.rho),
                               float(params.coherence_lambda), cap, N.ptr(fillshell),
                               N.ptr(enter), N.ptr(rows), cap + 1, N.ptr(report), N.ptr(ws),
                               ws_bytes, N.stream_ptr())
    if rc == N.GF_E_UNSUPPORTED:
        return run_coherence_fill_shells(u, lab0, params, tracked, order_log)
    N.check(rc)
    # one synchronisation: the report and the first rows in a single pinned copy
    head = min(cap + 1, 64)
    host = _pinned_report(4 + 10 * head)
    host[:4].copy_(report, non_blocking=True)
    host[4:].view(torch.int64).view(head, 5).copy_(rows[:head], non_blocking=True)
    torch.cuda.current_stream().synchronize()
    done, iters, deadlocks, filled = (int(v) for v in host[:4])
    if done == 3:
        raise N.NativeError("coherence fill: frontier capacity exceeded")
    r_h = host[4:].view(torch.int64).view(head, 5)[:iters] if iters <= head else rows[:iters].cpu()
    rep = dict(rows=[tuple(int(x) for x in r) for r in r_h.tolist()], iterations=iters,
               filled=filled, deadlock_fills=deadlocks, unfillable=done == 2, unfillable_count=0)
    if rep["unfillable"]:
        # the kernel leaves painting and the hull clip to the caller here
        from .engine import _paint_unfillable_device

        readable = lab0 == READABLE
        hull = None
        if bool(readable.any()):
            seed = u[readable]
            hull = (seed.min(), seed.max())
        rep["unfillable_count"] = _paint_unfillable_device(u, lab0, fillshell.reshape(H, W))
        if hull is not None:
            u.clamp_(hull[0], hull[1])
    rep["wall_time_s"] = time.perf_counter() - t0
    return u, rep, enter, fillshell


def run_coherence_fill_shells(u, lab0, params, tracked=True, order_log=False, g_at=None):
    """engine._fill_loop (engine.py:286-376) with one host-driven iteration per
    shell (the kernels of gf_coherence_directions, gf_sample_points,
    gf_commit_shell and gf_frontier_candidates).

    g comes from the masked structure tensor unless ``g_at(u, lab, frontier,
    pts)`` is given: it returns the frontier's (F, 2) float64 g and writes
    the pixels' (x, y) into ``pts`` (run_field_fill_shells: a guide field or a
    fixed g, for balls beyond the persistent kernels' tables).

    ``u``: (H, W, C) float64 CUDA tensor (consumed: filled in place); ``lab0``:
    (H, W) uint8 CUDA tensor (not modified).  Returns (u, report fields dict,
    enter, fillshell) with the order maps as int32 CUDA tensors (enter None
    unless order_log).
    """
    import torch

    H, W, C = u.shape
    dev = u.device
    lab = lab0.clone()
    flat_u = u.reshape(-1, C)
    flat_l = lab.reshape(-1)
    readable = lab == READABLE
    hull = None
    if bool(readable.any()):
        seed = u[readable]
        hull = (seed.min(), seed.max())
    remaining = int((lab == INPAINT).sum())
    data_term_live = params.order == "smart_with_data_term"
    px = bool(params.periodic_x)
    frontier = torch.nonzero(_active(lab, px)).reshape(-1)
    fillshell = torch.full((H * W,), -1, dtype=torch.int32, device=dev)
    enter = torch.full((H * W,), -1, dtype=torch.int32, device=dev) if order_log else None
    lib = N.load()
    if g_at is None:
        ws = torch.empty(lib.gf_coherence_workspace_bytes(H, W, C), dtype=torch.uint8, device=dev)

        def g_at(u_, lab_, fr, pts):
            return coherence_directions_device(u_, lab_, fr, params.sigma, params.rho,
                                               params.coherence_lambda, ws, pts)
    mark = torch.zeros(H * W, dtype=torch.uint8, device=dev)
    count = torch.zeros(1, dtype=torch.int32, device=dev)
    rep = dict(rows=[], iterations=0, filled=0, deadlock_fills=0, unfillable=False,
               unfillable_count=0)
    t0 = time.perf_counter()
    it = 0
    while remaining > 0:
        F = int(frontier.numel())
        if F == 0:
            rep["unfillable"] = True
            break
        if enter is not None:
            cur = enter[frontier]
            enter[frontier] = torch.where(cur < 0, torch.full_like(cur, it), cur)
        pts = torch.empty((F, 2), dtype=torch.float64, device=dev)
        g = g_at(u, lab, frontier, pts)
        rw, tw, vals = sample_points_device(u, lab, pts, g, params)
        if params.order == "onion":
            mode = 0
        elif params.order == "smart" or not data_term_live:
            mode = 1
        else:
            mode = 2
            if not bool((torch.hypot(g[:, 0], g[:, 1]) > 0.0).any()):
                data_term_live = False
                mode = 1
        count.zero_()
        fill = torch.empty(F, dtype=torch.uint8, device=dev)
        N.check(lib.gf_commit_shell(C, F, N.ptr(frontier), N.ptr(rw), N.ptr(tw), N.ptr(vals),
                                    N.ptr(g), mode, float(params.c), float(params.c2), it,
                                    N.ptr(u), N.ptr(lab), N.ptr(fillshell), N.ptr(fill),
                                    N.ptr(count), N.stream_ptr()))
        n = int(count.item())  # the shell's one synchronisation before the update
        if n == 0:
            # deadlock guard (engine.py:334-348): first maximal confidence, NaN first
            c_h = (rw / tw).cpu().numpy()
            k = int(np.argmax(c_h))
            if float(rw[k]) > 0.0:
                val = vals[k]
            else:
                val = _neighbor_mean(u, lab, int(frontier[k]), H, W, px)
                if val is None:
                    rep["unfillable"] = True
                    break
            p_k = frontier[k]
            flat_u[p_k] = val
            flat_l[p_k] = READABLE
            fillshell[p_k] = it
            fill[k] = 1
            n = 1
            rep["deadlock_fills"] += 1
        remaining -= n
        rep["filled"] += n
        if tracked:
            # tracker._update_arrays (tracker.py:59-79): survivors + Inpaint
            # neighbours of the filled pixels, sorted dedup, active filter
            mark.zero_()
            N.check(lib.gf_frontier_candidates(H, W, N.ptr(lab), 1 if px else 0, F,
                                               N.ptr(frontier), N.ptr(fill),
                                               N.ptr(mark), N.stream_ptr()))
            candidates = (mark != 0).sum()  # device scalar, read after the loop
            new_frontier = torch.nonzero(mark == 2).reshape(-1)
            threads = F
        else:
            new_frontier = torch.nonzero(_active(lab, px)).reshape(-1)
            candidates = threads = W * H
        rep["rows"].append((it, F, candidates, threads, n))
        frontier = new_frontier
        it += 1
    rep["iterations"] = it
    rep["rows"] = [(k, F, int(c), t, n) for (k, F, c, t, n) in rep["rows"]]
    if rep["unfillable"]:
        from .engine import _paint_unfillable_device

        rep["unfillable_count"] = _paint_unfillable_device(u, lab0, fillshell.reshape(H, W))
    if hull is not None:
        u.clamp_(hull[0], hull[1])
    rep["wall_time_s"] = time.perf_counter() - t0
    return u, rep, enter, fillshell


def run_field_fill_shells(u, lab0, params, field=None, tracked=True, order_log=False):
    """engine._fill_loop for a fixed or guide-field g (engine.py:234-242) through
    the shell-by-shell loop -- the path of balls with r > GF_MAX_RADIUS, whose
    sampler (gf_sample_points' large-ball kernel) keeps its tables in HBM.
    ``field``: (H, W, 2) float64 CUDA guide field, or None."""
    import torch

    H, W, _ = u.shape
    if params.g_source == "fixed":
        gf = params.g_fixed or (0.0, 0.0)
        const = torch.tensor([float(gf[0]), float(gf[1])], dtype=torch.float64, device=u.device)
    flat = field.reshape(-1, 2) if field is not None else None

    def g_at(u_, lab_, fr, pts):
        pts[:, 0] = (fr % W).to(torch.float64)
        pts[:, 1] = torch.div(fr, W, rounding_mode="floor").to(torch.float64)
        if params.g_source == "fixed":
            return const.expand(fr.numel(), 2).contiguous()
        if flat is None:
            return torch.zeros((fr.numel(), 2), dtype=torch.float64, device=u.device)
        return flat[fr].contiguous()

    return run_coherence_fill_shells(u, lab0, params, tracked, order_log, g_at=g_at)
