"""Device-level entry points: torch CUDA tensors in, torch CUDA tensors out.

These are thin wrappers around the C ABI (``_native``).  PyTorch provides
the device memory, the caching allocator and the current stream; all
compute happens in the sm_100a kernels of libgf_b200.so.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native as N


def params_to_c(params, tracked: bool, g_mode: int) -> N.FillParamsC:
    pc = N.FillParamsC()
    pc.r = int(params.r)
    pc.mu = float(params.mu)
    pc.c = float(params.c)
    pc.c2 = float(params.c2)
    pc.order = N.GF_ORDER[params.order]
    pc.neighborhood = N.GF_BALL[params.neighborhood]
    pc.g_mode = g_mode
    gf = params.g_fixed or (0.0, 0.0)
    pc.g_fixed[0] = float(gf[0])
    pc.g_fixed[1] = float(gf[1])
    pc.periodic_x = 1 if params.periodic_x else 0
    pc.tracked = 1 if tracked else 0
    return pc


def resolve_g_mode(params, guide_present: bool) -> int:
    """engine._resolve_g (engine.py:234-249) as a kernel mode."""
    if params.g_source == "fixed":
        return N.GF_G_FIXED
    if params.g_source == "guide_field":
        return N.GF_G_FIELD if guide_present else N.GF_G_ZERO
    raise NotImplementedError(
        "g_source='modified_structure_tensor' (coherence transport) recomputes g from the "
        "image every shell: it runs through engine.inpaint / tracker.run_tracked (the "
        "shell-by-shell loop of coherence.py), not the batched persistent kernel")


def _fill_setup(image, labels, guide, params, tracked=True, order_log=False, rows_cap=None,
                workspace=None, splines=None, eta=3.0, trace_cap=0, want_fillshell=False):
    """Output buffers, workspace and the C-ABI argument structs of one fill."""
    import torch

    N.require_cuda()
    lib = N.load()
    assert image.is_cuda and image.is_contiguous() and image.dim() == 4
    nF, H, W, C = image.shape
    # the kernels index labels as (nF, H, W) contiguous uint8 on the image's device
    if (tuple(labels.shape[-2:]) != (H, W) or labels.dtype != torch.uint8 or not labels.is_cuda
            or not labels.is_contiguous() or labels.numel() not in (H * W, nF * H * W)):
        raise ValueError("image and label shapes differ")
    if labels.numel() != nF * H * W:
        raise ValueError(f"{labels.numel() // (H * W)} label masks for {nF} frames")
    raster = splines is not None and splines.n_seg > 0
    g_mode = N.GF_G_FIELD if raster else resolve_g_mode(params, guide is not None)
    if g_mode != N.GF_G_FIELD or raster:
        guide = None
    dev = image.device
    dtype = N.GF_F64 if image.dtype == torch.float64 else N.GF_F32
    out = torch.empty_like(image)
    stats = torch.empty((nF, N.GF_STATS), dtype=torch.int32, device=dev)  # every field is written
    if rows_cap is None:
        rows_cap = min(H * W + 1, max(1024, (1 << 24) // max(1, nF)))
    rows = torch.empty((nF, rows_cap, 2), dtype=torch.int32, device=dev)
    enter = fillshell = None
    if order_log:
        enter = torch.empty((nF, H, W), dtype=torch.int32, device=dev)
    if order_log or want_fillshell:
        fillshell = torch.empty((nF, H, W), dtype=torch.int32, device=dev)
    fr = N.FramesC(nF, H, W, C, dtype, image.data_ptr(), labels.data_ptr(),
                   0 if guide is None else guide.data_ptr(), out.data_ptr())
    pc = params_to_c(params, tracked, g_mode)
    trace = None
    if trace_cap:
        trace = torch.zeros((trace_cap, 8), dtype=torch.int64, device=dev)
    oc = N.FillOutputsC(stats.data_ptr(), rows.data_ptr(), rows_cap,
                        0 if enter is None else enter.data_ptr(),
                        0 if fillshell is None else fillshell.data_ptr(),
                        0 if trace is None else trace.data_ptr(), int(trace_cap))
    sc = splines.as_c(eta) if raster else None
    if raster:
        need = lib.gf_fill_splines_workspace_bytes(ctypes.byref(fr), ctypes.byref(pc),
                                                   ctypes.byref(sc))
    else:
        need = lib.gf_fill_workspace_bytes(ctypes.byref(fr), ctypes.byref(pc))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    res = dict(out=out, stats=stats, rows=rows, enter=enter, fillshell=fillshell,
               workspace=workspace, rows_cap=rows_cap, trace=trace)
    # the structs keep raw pointers: hold the tensors they point into
    call = dict(fr=fr, pc=pc, oc=oc, sc=sc, need=need, keep=(image, labels, guide, splines))
    return res, call


def _fill_launch(res, call):
    """The C-ABI fill call on the current stream (memset + k_prep + k_shells)."""
    lib = N.load()
    ws = ctypes.c_void_p(res["workspace"].data_ptr())
    if call["sc"] is not None:
        N.check(lib.gf_fill_splines(ctypes.byref(call["fr"]), ctypes.byref(call["pc"]),
                                    ctypes.byref(call["sc"]), ctypes.byref(call["oc"]), ws,
                                    call["need"], N.stream_ptr()))
    else:
        N.check(lib.gf_fill(ctypes.byref(call["fr"]), ctypes.byref(call["pc"]),
                            ctypes.byref(call["oc"]), ws, call["need"], N.stream_ptr()))


def fill_device(image, labels, guide, params, tracked=True, order_log=False, rows_cap=None,
                workspace=None, splines=None, eta=3.0, trace_cap=0, want_fillshell=False):
    """Fill a batch of frames on the GPU.

    image: (N, H, W, C) float32/float64 CUDA tensor; labels: (N, H, W) uint8;
    guide: (N, H, W, 2) float64 or None; splines: a SegmentSet to raster the
    guide field inside the fill (gf_fill_splines) instead of ``guide``.
    Returns a dict of CUDA tensors: ``out`` (like image), ``stats``
    (N, GF_STATS) int32, ``rows`` (N, rows_cap, 2) int32, with order_log
    ``enter``/``fillshell`` (N, H, W) int32, with trace_cap > 0 ``trace``
    (trace_cap, 8) int64 per-shell phase timestamps.
    """
    res, call = _fill_setup(image, labels, guide, params, tracked, order_log, rows_cap, workspace,
                            splines, eta, trace_cap, want_fillshell)
    _fill_launch(res, call)
    return res


class FillGraph:
    """One fill captured as a CUDA graph for fixed device buffers.

    For streams of same-shaped frames (video, serving): the memset, k_prep
    and the cooperative shell kernel replay without any host launch work.
    New frames are written into the ``image`` / ``labels`` tensors given
    here (``copy_``); ``replay()`` refills ``self.res`` (the fill_device
    outputs) on the current stream.
    """

    def __init__(self, image, labels, guide, params, tracked=True, rows_cap=4096, splines=None,
                 eta=3.0, want_fillshell=False):
        import torch

        self.res, self.call = _fill_setup(image, labels, guide, params, tracked, False, rows_cap,
                                          None, splines, eta, 0, want_fillshell)
        _fill_launch(self.res, self.call)  # warm-up: function attributes, occupancy
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        n0 = N.launch_count()
        with torch.cuda.graph(self.graph):
            _fill_launch(self.res, self.call)
        # kernels of the library inside the graph: what every replay launches
        self.launches_per_replay = N.launch_count() - n0
        torch.cuda.synchronize()

    def replay(self):
        self.graph.replay()
        return self.res


class BatchGraph:
    """A video block filled in chunks of frames, captured as ONE CUDA graph.

    images (N, H, W, C) / labels (N, H, W) CUDA tensors; ``splines``: one
    Spline list per frame (rastered inside each fill).  Chunk c fills frames
    [c*chunk, (c+1)*chunk) with one batched gf_fill_splines call; the chunks
    run back to back on one stream and share one workspace.  ``replay()``
    refills every chunk's result dict (``self.parts``).
    """

    def __init__(self, images, labels, splines, params, chunk=64, tracked=True, rows_cap=4096,
                 eta=3.0, streams=1):
        import torch

        n = images.shape[0]
        self.parts = []
        calls = []
        wss = [None] * streams
        for k, c0 in enumerate(range(0, n, chunk)):
            c1 = min(n, c0 + chunk)
            segs = SegmentSet(list(splines[c0:c1]), images.device, per_frame=True)
            res, call = _fill_setup(images[c0:c1], labels[c0:c1], None, params, tracked, False,
                                    rows_cap, wss[k % streams], segs, eta, 0, False)
            wss[k % streams] = res["workspace"]  # one workspace per stream
            res["frames"] = (c0, c1)
            self.parts.append(res)
            calls.append(call)
        for res, call in zip(self.parts, calls):
            _fill_launch(res, call)
        torch.cuda.synchronize()
        self.calls = calls
        self.graph = torch.cuda.CUDAGraph()
        n0 = N.launch_count()
        with torch.cuda.graph(self.graph):
            if streams == 1:
                for res, call in zip(self.parts, calls):
                    _fill_launch(res, call)
            else:
                # chunks alternate over forked streams: chunk k+1's prep can run
                # beside chunk k's shell loop (each stream reuses its workspace)
                main = torch.cuda.current_stream()
                side = [torch.cuda.Stream() for _ in range(streams)]
                for st in side:
                    st.wait_stream(main)
                for k, (res, call) in enumerate(zip(self.parts, calls)):
                    with torch.cuda.stream(side[k % streams]):
                        _fill_launch(res, call)
                for st in side:
                    main.wait_stream(st)
        self.launches_per_replay = N.launch_count() - n0
        torch.cuda.synchronize()

    def replay(self):
        self.graph.replay()
        return self.parts

    def stats(self):
        import torch

        return torch.cat([p["stats"] for p in self.parts]).cpu().numpy()


def splines_to_segments(splines):
    """Host-side polyline flattening (splines.py:42-73) -> segment arrays."""
    segs, owner, dirs = [], [], []
    for s_idx, sp in enumerate(splines):
        poly = np.asarray(sp.polyline(), dtype=np.float64)
        for k in range(len(poly) - 1):
            segs.append((poly[k, 0], poly[k, 1], poly[k + 1, 0], poly[k + 1, 1]))
            owner.append(s_idx)
        dirs.append((float(sp.direction[0]), float(sp.direction[1])))
    seg = np.asarray(segs, dtype=np.float64).reshape(-1, 4)
    own = np.asarray(owner, dtype=np.int32)
    dv = np.asarray(dirs, dtype=np.float64).reshape(-1, 2)
    return seg, own, dv


class SegmentSet:
    """Flattened splines resident on the device (reused across steps).

    ``splines`` is one spline list shared by every frame, or, with
    ``per_frame=True``, a list of spline lists (one per frame of a batch).
    """

    def __init__(self, splines, device, per_frame=False):
        import torch

        if per_frame:
            segs, owns, dirs, offs = [], [], [], [0]
            base = 0
            for frame_splines in splines:
                seg, own, dv = splines_to_segments(list(frame_splines))
                segs.append(seg)
                owns.append(own + base)
                dirs.append(dv)
                base += len(dv)
                offs.append(offs[-1] + len(seg))
            seg = np.concatenate(segs) if segs else np.zeros((0, 4))
            own = np.concatenate(owns).astype(np.int32) if owns else np.zeros(0, np.int32)
            dv = np.concatenate(dirs) if dirs else np.zeros((0, 2))
            self.frame_seg = torch.tensor(offs, dtype=torch.int32, device=device)
        else:
            seg, own, dv = splines_to_segments(list(splines))
            self.frame_seg = None
        self.n_splines = len(dv)
        self.n_seg = len(seg)
        self.seg = torch.from_numpy(np.ascontiguousarray(seg)).to(device)
        self.owner = torch.from_numpy(np.ascontiguousarray(own, dtype=np.int32)).to(device)
        self.dirs = torch.from_numpy(np.ascontiguousarray(dv)).to(device)

    _cache = {}
    _cache_order = []

    @classmethod
    def cached(cls, splines, device, max_entries=64):
        """A SegmentSet for ``splines`` reused across calls: keyed on the
        splines' content (control points, kind, direction), so repeated
        fills with the same guide curves skip the host flattening and upload."""
        key = (str(device), tuple((tuple(np.asarray(s.points, dtype=np.float64).ravel().tolist()),
                                   str(getattr(s, "kind", "")),
                                   tuple(np.asarray(s.direction, dtype=np.float64).tolist()))
                                  for s in splines))
        hit = cls._cache.get(key)
        if hit is not None:
            return hit
        seg = cls(splines, device)
        cls._cache[key] = seg
        cls._cache_order.append(key)
        if len(cls._cache_order) > max_entries:
            cls._cache.pop(cls._cache_order.pop(0), None)
        return seg

    def as_c(self, eta=3.0):
        return N.SplinesC(self.n_seg, self.seg.data_ptr(), self.owner.data_ptr(), self.n_splines,
                          self.dirs.data_ptr(), float(eta),
                          0 if self.frame_seg is None else self.frame_seg.data_ptr())


def guide_field_device(labels, segset: SegmentSet, eta: float = 3.0, out=None):
    """(H, W) uint8 CUDA labels -> (H, W, 2) float64 CUDA guide field."""
    import torch

    N.require_cuda()
    lib = N.load()
    H, W = labels.shape[-2:]
    if out is None:
        out = torch.empty((H, W, 2), dtype=torch.float64, device=labels.device)
    N.check(lib.gf_guide_field(H, W, N.ptr(labels), segset.n_seg, N.ptr(segset.seg),
                               N.ptr(segset.owner), segset.n_splines, N.ptr(segset.dirs),
                               float(eta), N.ptr(out), N.stream_ptr()))
    return out


def sample_points_device(image, labels, points, g, params):
    """Ball sampler at points: (rw, tw, vals) CUDA tensors."""
    import torch

    N.require_cuda()
    lib = N.load()
    H, W, C = image.shape
    n = points.shape[0]
    rw = torch.empty(n, dtype=torch.float64, device=image.device)
    tw = torch.empty(n, dtype=torch.float64, device=image.device)
    vals = torch.empty((n, C), dtype=torch.float64, device=image.device)
    pc = params_to_c(params, True, N.GF_G_FIELD)
    N.check(lib.gf_sample_points(H, W, C, N.ptr(image), N.ptr(labels), n, N.ptr(points), N.ptr(g),
                                 ctypes.byref(pc), N.ptr(rw), N.ptr(tw), N.ptr(vals),
                                 N.stream_ptr()))
    return rw, tw, vals


def bilinear_device(image, labels, X, Y, periodic_x):
    import torch

    N.require_cuda()
    lib = N.load()
    H, W, C = image.shape
    n = X.numel()
    vals = torch.empty((n, C), dtype=torch.float64, device=image.device)
    ok = torch.empty(n, dtype=torch.uint8, device=image.device)
    N.check(lib.gf_bilinear_gather(H, W, C, N.ptr(image), N.ptr(labels), n, N.ptr(X), N.ptr(Y),
                                   1 if periodic_x else 0, N.ptr(vals), N.ptr(ok), N.stream_ptr()))
    return vals, ok


def boundary_device(labels, periodic_x):
    import torch

    N.require_cuda()
    lib = N.load()
    H, W = labels.shape
    act = torch.empty((H, W), dtype=torch.uint8, device=labels.device)
    inn = torch.empty_like(act)
    out = torch.empty_like(act)
    N.check(lib.gf_boundary_masks(H, W, N.ptr(labels), 1 if periodic_x else 0, N.ptr(act),
                                  N.ptr(inn), N.ptr(out), N.stream_ptr()))
    return act, inn, out
