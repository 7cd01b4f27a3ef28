"""Shell-based Guidefill fill engine -- drop-in for the reference engine.py.

Same public surface as /root/reference/pkg/src/guidefill/engine.py:
``FillParams`` (engine.py:33-91), ``FillReport`` (:94-115), ``weight``
(:118-128), ``confidence`` / ``fill_color`` (:202-221), ``ready``
(:224-231) and ``inpaint`` (:379-408), with the same argument meaning,
return layout and ValueError messages.  The fill itself runs on the GPU:
``_run_fill`` hands the frame to the persistent sm_100a shell kernel through
the C ABI (gf_fill) and only copies the result back.

The unfillable fallback (engine.py:270-283) runs on the device too: when the
frontier empties while Inpaint pixels remain (a Bystander moat), the
stranded pixels take the colour of the nearest readable pixel, found by
gf_paint_unfillable -- a restatement of scipy's Euclidean distance-transform
feature transform with its tie-breaking (csrc/gf_unfill.cu).
"""

from __future__ import annotations

import math
import time
from dataclasses import asdict, dataclass, field

import numpy as np

from . import _native as N
from . import grid
from .grid import INPAINT, READABLE

ORDERS = ("onion", "smart", "smart_with_data_term")
NEIGHBORHOODS = ("rotated_ball", "axis_ball")
G_SOURCES = ("guide_field", "modified_structure_tensor", "fixed")


@dataclass
class FillParams:
    """Knobs of the fill engine; defaults are the guide-field configuration."""

    r: int = 3
    mu: float = 50.0
    c: float = 0.05
    c2: float = 0.0
    order: str = "smart"
    neighborhood: str = "rotated_ball"
    g_source: str = "guide_field"
    g_fixed: tuple | None = None
    periodic_x: bool = False
    sigma: float = 2.0
    rho: float = 4.0
    coherence_lambda: float = 1e-5

    def __post_init__(self):
        if self.r < 1:
            raise ValueError("r must be >= 1")
        if self.order not in ORDERS:
            raise ValueError(f"order must be one of {ORDERS}")
        if self.neighborhood not in NEIGHBORHOODS:
            raise ValueError(f"neighborhood must be one of {NEIGHBORHOODS}")
        if self.g_source not in G_SOURCES:
            raise ValueError(f"g_source must be one of {G_SOURCES}")
        if not (self.mu >= 0.0):
            raise ValueError("mu must be >= 0 (inf allowed)")

    @classmethod
    def guidefill(cls, **kw) -> "FillParams":
        return cls(**kw)

    @classmethod
    def coherence_transport(cls, **kw) -> "FillParams":
        """Axis-ball transport steered by the boundary-aware structure tensor."""
        defaults = dict(r=5, neighborhood="axis_ball", order="onion",
                        g_source="modified_structure_tensor")
        defaults.update(kw)
        return cls(**defaults)

    @classmethod
    def telea(cls, **kw) -> "FillParams":
        """Isotropic onion baseline: axis ball, g = 0."""
        defaults = dict(neighborhood="axis_ball", order="onion", g_source="fixed",
                        g_fixed=(0.0, 0.0))
        defaults.update(kw)
        return cls(**defaults)

    def to_dict(self) -> dict:
        d = asdict(self)
        if math.isinf(d["mu"]):
            d["mu"] = "inf"
        return d


@dataclass
class FillReport:
    iterations: int = 0
    filled: int = 0
    deadlock_fills: int = 0
    unfillable: bool = False
    unfillable_count: int = 0
    wall_time_s: float = 0.0
    # per-iteration rows: (iteration, frontier_size, candidates, threads_requested, filled)
    rows: list = field(default_factory=list)

    def to_dict(self) -> dict:
        return {
            "iterations": self.iterations,
            "filled": self.filled,
            "deadlock_fills": self.deadlock_fills,
            "unfillable": self.unfillable,
            "unfillable_count": self.unfillable_count,
            "wall_time_s": self.wall_time_s,
            "frontier_sizes": [r[1] for r in self.rows],
            "filled_per_iteration": [r[4] for r in self.rows],
        }


def weight(x, y, g, mu: float, eps: float) -> float:
    """Pairwise Eq. 3.2 weight for finite mu (engine.py:118-128); host scalar."""
    dx = float(y[0]) - float(x[0])
    dy = float(y[1]) - float(x[1])
    dist = math.hypot(dx, dy)
    if dist == 0.0:
        raise ValueError("weight is undefined at y == x")
    if math.isinf(mu):
        raise ValueError("mu = inf weights are defined set-wise, not pairwise")
    d = -float(g[1]) * dx + float(g[0]) * dy
    return math.exp(-(mu * mu) / (2.0 * eps * eps) * d * d) / dist


def _point_gather(point, image, labels, g, params):
    import torch

    dev = N.require_cuda()
    from ._device import sample_points_device

    img = np.ascontiguousarray(image, dtype=np.float64)
    lab = np.ascontiguousarray(np.where(np.asarray(labels) == READABLE, READABLE, grid.BYSTANDER),
                               dtype=np.uint8)
    pts = torch.tensor([[float(point[0]), float(point[1])]], dtype=torch.float64, device=dev)
    gv = np.asarray(g, dtype=np.float64).reshape(1, 2)
    rw, tw, vals = sample_points_device(torch.from_numpy(img).to(dev), torch.from_numpy(lab).to(dev),
                                        pts, torch.from_numpy(gv).to(dev), params)
    return vals.cpu().numpy(), rw.cpu().numpy(), tw.cpu().numpy()



def confidence(point, image, labels, g, params: FillParams) -> float:
    """Readable over total ball weight mass at one pixel (Eq. 3.7, engine.py:202-209)."""
    _, rw, tw = _point_gather(point, image, labels, g, params)
    return float(rw[0] / tw[0])


def fill_color(point, image, labels, g, params: FillParams):
    """Weighted average of readable ball samples; (values, True) or (None, False)."""
    vals, rw, _ = _point_gather(point, image, labels, g, params)
    if rw[0] == 0.0:
        return None, False
    return vals[0], True


def ready(conf: float, g, params: FillParams, data_term_live: bool = True) -> bool:
    """Fill-readiness predicate for one pixel (engine.py:224-231)."""
    if params.order == "onion":
        return True
    if params.order == "smart" or not data_term_live:
        return conf > params.c
    gnorm = math.hypot(float(g[0]), float(g[1]))
    return gnorm > params.c2 and conf > params.c


def _paint_unfillable_device(out, labels_dev, fillshell_dev):
    """Stranded Inpaint pixels take their nearest readable colour on the
    device (engine.py:270-283 via gf_paint_unfillable: scipy's EDT feature
    transform restated, ties included).  out (H, W, C) CUDA tensor, in place.
    Returns the painted pixel count (synchronises)."""
    import torch

    lib = N.load()
    H, W, C = out.shape
    need = lib.gf_paint_unfillable_workspace_bytes(H, W)
    ws = torch.empty(need, dtype=torch.uint8, device=out.device)
    cnt = torch.zeros(1, dtype=torch.int32, device=out.device)
    N.check(lib.gf_paint_unfillable(H, W, C, N.GF_F64 if out.dtype == torch.float64 else N.GF_F32,
                                    N.ptr(labels_dev), N.ptr(fillshell_dev), N.ptr(out), N.ptr(ws),
                                    need, N.ptr(cnt), N.stream_ptr()))
    return int(cnt.item())


def _is_spline_list(guide) -> bool:
    return isinstance(guide, (list, tuple)) and all(hasattr(s, "polyline") for s in guide)


def _report_from(stats, rows_dev, tracked: bool, H: int, W: int) -> FillReport:
    """FillReport of one frame from its device stats and (F, filled) rows."""
    iters = int(stats[N.STAT_ITERATIONS])
    rep = FillReport()
    rep.iterations = iters
    rep.filled = int(stats[N.STAT_FILLED])
    rep.deadlock_fills = int(stats[N.STAT_DEADLOCK])
    rows = []
    for k in range(iters):
        F, filled = int(rows_dev[k, 0]), int(rows_dev[k, 1])
        if tracked:
            # candidates == next frontier size (the active filter never
            # removes a candidate)
            cand = int(rows_dev[k + 1, 0]) if k + 1 < iters else int(stats[N.STAT_LAST_FRONTIER])
            rows.append((k, F, cand, F, filled))
        else:
            rows.append((k, F, W * H, W * H, filled))
    rep.rows = rows
    return rep


def _run_fill(image, labels, guide_vecs, params: FillParams, tracked: bool, order_log=False,
              splines=None, eta=3.0, validate=False):
    """Fill one frame on the GPU.  Returns (u float64 (H,W,C), FillReport, maps).

    ``splines`` (a list of Spline) rasters the guide field inside the fill
    (gf_fill_splines) instead of uploading a dense ``guide_vecs``.
    """
    import torch

    if validate and not torch.cuda.is_available():
        grid.validate_labels(labels)  # same ValueError without a device
    dev = N.require_cuda()
    if params.g_source == "modified_structure_tensor":
        return _run_coherence(image, labels, params, tracked, order_log, dev)
    if params.r > N.GF_MAX_RADIUS:
        return _run_large_ball(image, labels, guide_vecs, params, tracked, order_log, dev,
                               splines, eta)
    from . import _staging
    from ._device import SegmentSet, fill_device

    H, W = labels.shape
    # torch tensors (CPU -- pinned ones are DMA'd straight from the caller's
    # memory -- or CUDA) are accepted next to the reference's numpy arrays;
    # the result comes back in the caller's kind (numpy f64 / CPU tensor)
    as_tensor = isinstance(image, torch.Tensor)
    t0 = time.perf_counter()
    if isinstance(labels, torch.Tensor):
        d_lab = labels.to(torch.uint8).to(dev, non_blocking=labels.is_pinned()).reshape(1, H, W)
        labels = labels.cpu().numpy() if labels.is_cuda else labels.numpy()
    else:
        # labels first (small, direct), then the image through the chunked
        # pinned stager; the spline segments come from a content-keyed cache
        d_lab = torch.from_numpy(np.ascontiguousarray(labels, dtype=np.uint8)).to(dev).reshape(1, H, W)
    d_guide = None
    segs = None
    if splines is not None and params.g_source == "guide_field":
        segs = SegmentSet.cached(list(splines), dev) if len(splines) else None
    mirror = None
    if as_tensor:
        timg = image.to(torch.float64).contiguous()
        C = timg.shape[2]
        if (not timg.is_cuda and timg.is_pinned() and timg.numel() * 8 >= (1 << 20)
                and _staging.mirror_supported(dev)):
            d_img, mirror = _staging.upload_mirrored(timg, dev, True)
            d_img = d_img.reshape(1, H, W, C)
        else:
            d_img = (timg if timg.is_cuda else timg.to(dev, non_blocking=timg.is_pinned())).reshape(1, H, W, C)
    else:
        img = np.ascontiguousarray(image, dtype=np.float64)
        C = img.shape[2]
        if img.nbytes >= (1 << 20) and _staging.mirror_supported(dev):
            d_img, mirror = _staging.upload_mirrored(img, dev, False)
            d_img = d_img.reshape(1, H, W, C)
        else:
            d_img = _staging.upload(img, dev, "img").reshape(1, H, W, C)
    if guide_vecs is not None and params.g_source == "guide_field" and segs is None:
        d_guide = _staging.upload(np.ascontiguousarray(guide_vecs, dtype=np.float64), dev,
                                  "guide").reshape(1, H, W, 2)
    try:
        res = fill_device(d_img, d_lab, d_guide, params, tracked=tracked, order_log=order_log,
                          rows_cap=H * W + 1, splines=segs, eta=eta, want_fillshell=True)
        if mirror is not None:
            # result = the mirrored input + the changed pixels (the read-back of
            # the report below synchronises the stream)
            mirror.finish(d_img, res["out"])
        stats, rows_dev = _staging.read_report(res["stats"][0], res["rows"][0])
    except BaseException:
        if mirror is not None:
            # the mirror DMA still targets the pooled result buffer: let it land
            # before the buffer can be handed to another caller
            mirror.settle()
        raise
    if validate and stats[N.STAT_BAD_LABELS]:
        grid.validate_labels(labels)  # k_prep saw a bad label: the reference's message
        raise ValueError("label mask holds values outside {0, 128, 255}")
    iters = int(stats[N.STAT_ITERATIONS])
    n_painted = 0
    if stats[N.STAT_UNFILLABLE]:
        # stranded pixels: painted on the device before the result leaves it
        n_painted = _paint_unfillable_device(res["out"][0], d_lab[0], res["fillshell"][0])
        if mirror is not None:
            mirror.finish(d_img, res["out"])  # the painted pixels join the delta
    if iters + 1 > rows_dev.shape[0]:
        rows_dev = res["rows"][0, :iters + 1].cpu().numpy()
    if mirror is not None:
        torch.cuda.current_stream().synchronize()  # the delta has landed
        if as_tensor:
            u_t = mirror.result
        else:
            u = mirror.result
    elif as_tensor:
        u_t = _staging.download_tensor(res["out"][0])
    else:
        u = _staging.download(res["out"][0])
    rep = _report_from(stats, rows_dev, tracked, H, W)
    fillshell = None
    if order_log or stats[N.STAT_UNFILLABLE]:
        fillshell = res["fillshell"][0].cpu().numpy()
    if stats[N.STAT_UNFILLABLE]:
        rep.unfillable = True
        rep.unfillable_count = n_painted
        fillshell = np.where((np.asarray(labels) == INPAINT) & (fillshell < 0), -2, fillshell)
    enter = res["enter"][0].cpu().numpy() if order_log else None
    rep.wall_time_s = time.perf_counter() - t0
    return (u_t if as_tensor else u), rep, dict(enter=enter, fillshell=fillshell)


def _run_large_ball(image, labels, guide_vecs, params, tracked, order_log, dev, splines, eta):
    """Balls with r > GF_MAX_RADIUS (the reference takes any r >= 1,
    engine.py:51-52): the shell-by-shell device loop with the large-ball
    sampler (coherence.run_field_fill_shells).  Same return layout as _run_fill."""
    import torch

    from ._device import SegmentSet, guide_field_device
    from .coherence import run_field_fill_shells

    def runner(work, d_lab):
        field = None
        if params.g_source == "guide_field":
            if splines is not None:
                segs = SegmentSet.cached(list(splines), dev) if len(splines) else None
                if segs is not None:
                    field = guide_field_device(d_lab, segs, eta)
            elif guide_vecs is not None:
                field = torch.from_numpy(np.ascontiguousarray(guide_vecs, dtype=np.float64)).to(dev)
        return run_field_fill_shells(work, d_lab, params, field, tracked, order_log)

    return _run_coherence(image, labels, params, tracked, order_log, dev, runner)


def _run_coherence(image, labels, params, tracked, order_log, dev, runner=None):
    """Coherence-transport g source (engine.py:243-249): the one-launch device loop
    of coherence.run_coherence_fill (or ``runner(work, d_lab)``, the large-ball
    loop).  Same return layout as _run_fill; host frames travel like _run_fill's
    (chunked pinned upload mirrored back into the result buffer, then only the
    changed pixels come down)."""
    import torch

    from . import _staging
    from .coherence import run_coherence_fill

    if runner is None:
        def runner(work, d_lab):
            return run_coherence_fill(work, d_lab, params, tracked, order_log)
    t0 = time.perf_counter()
    as_tensor = isinstance(image, torch.Tensor)
    if isinstance(labels, torch.Tensor):
        labels = labels.cpu().numpy()
    lab_np = np.ascontiguousarray(labels, dtype=np.uint8)
    H, W = lab_np.shape
    d_lab = torch.from_numpy(lab_np).to(dev)
    bad = (d_lab != READABLE) & (d_lab != grid.BYSTANDER) & (d_lab != INPAINT)
    if bool(bad.any()):
        grid.validate_labels(labels)
        raise ValueError("label mask holds values outside {0, 128, 255}")
    mirror = None
    if as_tensor:
        timg = image.to(torch.float64).contiguous()
        if (not timg.is_cuda and timg.is_pinned() and timg.numel() * 8 >= (1 << 20)
                and _staging.mirror_supported(dev)):
            d_img, mirror = _staging.upload_mirrored(timg, dev, True)
        else:
            d_img = timg.to(dev, non_blocking=timg.is_pinned())
    else:
        img = np.ascontiguousarray(image, dtype=np.float64)
        if img.nbytes >= (1 << 20) and _staging.mirror_supported(dev):
            d_img, mirror = _staging.upload_mirrored(img, dev, False)
        else:
            d_img = _staging.upload(img, dev, "img")
    # the fill works in place: keep the input (the caller's tensor, or the
    # delta's reference) intact
    aliased = as_tensor and image.is_cuda and d_img.data_ptr() == image.data_ptr()
    work = d_img.clone() if (mirror is not None or aliased) else d_img
    try:
        u, r, enter, fillshell = runner(work, d_lab)
        if mirror is not None:
            mirror.finish(d_img, u)
            torch.cuda.current_stream().synchronize()
    except BaseException:
        if mirror is not None:
            mirror.settle()
        raise
    rep = FillReport()
    rep.iterations = r["iterations"]
    rep.filled = r["filled"]
    rep.deadlock_fills = r["deadlock_fills"]
    rep.unfillable = r["unfillable"]
    rep.unfillable_count = r["unfillable_count"]
    rep.rows = r["rows"]
    if mirror is not None:
        out = mirror.result
    else:
        out = u.cpu() if as_tensor else u.cpu().numpy()
    fs = None
    if order_log or rep.unfillable:
        fs = fillshell.reshape(H, W).cpu().numpy()
        if rep.unfillable:
            fs = np.where((lab_np == INPAINT) & (fs < 0), -2, fs)
    en = enter.reshape(H, W).cpu().numpy() if enter is not None else None
    rep.wall_time_s = time.perf_counter() - t0
    return out, rep, dict(enter=en, fillshell=fs)


class FrontierRuleError(NotImplementedError):
    """A frontier_update hook returned a frontier other than the tracker's."""


def _shell_sets(enter, fillshell, iterations):
    """Per-shell sorted frontiers and fill masks from the engine's order log
    (frontier(k) = {p : enter[p] <= k <= fillshell[p]}, never-filled pixels
    stay until the end): yields (k, frontier, fill)."""
    enter = np.asarray(enter).reshape(-1)
    fs = np.asarray(fillshell).reshape(-1)
    members = np.flatnonzero(enter >= 0)
    start = enter[members]
    stop = np.where(fs[members] >= 0, fs[members], iterations)
    order_in = np.argsort(start, kind="stable")
    order_out = np.argsort(stop, kind="stable")
    cur = np.empty(0, dtype=np.int64)
    a = b = 0
    for k in range(iterations):
        lo = a
        while a < members.size and start[order_in[a]] <= k:
            a += 1
        if a > lo:
            cur = np.union1d(cur, members[order_in[lo:a]])
        lo = b
        while b < members.size and stop[order_out[b]] < k:
            b += 1
        if b > lo:
            cur = np.setdiff1d(cur, members[order_out[lo:b]], assume_unique=True)
        yield k, cur, fs[cur] == k


def _fill_loop(image, labels, guide_vecs, params: FillParams, frontier_update=None):
    """The reference's fill seam (engine.py:286-376): (u, lab, report).

    This is the one function every reference caller goes through (inpaint,
    run_tracked and their callers), so routing ``guidefill.engine._fill_loop``
    here reroutes them to the device.  The shell loop itself
    runs in the persistent kernel; a ``frontier_update`` hook is replayed
    afterwards from the kernel's order log, one call per shell with exactly
    the arguments the reference passes (sorted frontier, fill mask, filled
    indices, labels relabelled so far).  The hook's candidate counts go into
    the report rows as in the reference; a hook that returns a frontier other
    than the tracker's (a custom rule the device loop cannot follow) raises
    FrontierRuleError.
    """
    tracked = frontier_update is not None
    u, report, maps = _run_fill(image, labels, guide_vecs, params, tracked=tracked,
                                order_log=tracked, validate=True)
    lab = np.array(labels, dtype=np.uint8, copy=True)
    if not tracked:
        lab[lab == INPAINT] = READABLE
        return u, lab, report
    flat = lab.reshape(-1)
    nxt = None
    rows = []
    for k, frontier, fill in _shell_sets(maps["enter"], maps["fillshell"], report.iterations):
        if nxt is not None and not np.array_equal(nxt, frontier):
            raise FrontierRuleError("the frontier_update hook returned a frontier other than the "
                                    "tracked update's; custom frontier rules are not supported")
        filled_idx = frontier[fill]
        flat[filled_idx] = READABLE
        candidates, new_frontier = frontier_update(frontier, fill, filled_idx, lab)
        nxt = np.asarray(new_frontier, dtype=np.int64)
        rows.append((k, int(frontier.size), int(candidates), int(frontier.size),
                     int(filled_idx.size)))
    if report.iterations and nxt.size and not report.unfillable:
        raise FrontierRuleError("the frontier_update hook kept pixels after the last shell")
    report.rows = rows
    lab[lab == INPAINT] = READABLE  # painted (unfillable fallback) pixels too
    return u, lab, report


def inpaint(image, labels, guide=None, params: FillParams | None = None):
    """Fill all Inpaint pixels of ``labels`` in ``image`` (engine.py:379-408).

    Untracked variant: the GPU rescans the whole lattice for the frontier
    after every shell (threads = W*H), like the reference's plain loop.
    Returns (filled_image float64 (H, W, C), FillReport).
    """
    params = params or FillParams()
    labels = np.asarray(labels)
    if labels.ndim != 2:
        grid.validate_labels(labels)
    if labels.dtype != np.uint8:
        grid.validate_labels(labels)  # values are scanned on the GPU for uint8 masks
    if image.ndim != 3:
        raise ValueError("image must be (H, W, C)")
    if image.shape[:2] != labels.shape:
        raise ValueError(
            f"image {image.shape[:2]} and label mask {labels.shape} dimensions differ"
        )
    if _is_spline_list(guide):
        # extension: splines instead of a field -> rastered inside the fill
        u, report, _ = _run_fill(image, labels, None, params, tracked=False, splines=guide,
                                 validate=True)
        return u, report
    guide_vecs = None
    if guide is not None:
        guide_vecs = np.asarray(guide, dtype=np.float64)
        if guide_vecs.shape != labels.shape + (2,):
            raise ValueError("guide field shape must be (H, W, 2)")
    u, report, _ = _run_fill(image, labels, guide_vecs, params, tracked=False, validate=True)
    return u, report


def coherence_transport_mode(image, labels, **param_overrides):
    """engine.py:411-414: coherence transport (masked structure-tensor g, axis ball, onion)."""
    params = FillParams.coherence_transport(**param_overrides)
    return inpaint(image, labels, None, params)
