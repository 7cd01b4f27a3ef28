"""Complexity studies on the GPU: the paper's T(N) / P(N) experiment.

The reference's ``harness`` module (pkg/src/guidefill/harness.py) renders
two-tone continuum problems at a family of resolutions and fits power laws
to fill time and lane demand.  This is the paper's Section 6 figure (PAPER.md,
"Experimental time complexity T(N) and processor complexity P(N)"):
alpha = 0.54 / 1.10 and beta = 0.5 / 1.0 with / without tracking.

Here the same study runs on the B200 engine, rendered straight into device
memory, so the resolution sweep reaches 1e8 px:
- ``SyntheticProblem``, ``pixel_centers``, ``render_problem`` follow
  harness.py:27-47, 86-127 (same fields, same rasterisation: hard threshold
  at pixel centres, fp64 with numpy's operation order);
- ``render_problem_device`` produces the identical arrays with torch on the
  GPU (elementwise fp64, one op per kernel, so no contraction);
- ``scaling_study`` follows harness.py:277-306 (same defaults, same row keys),
  with ``seconds`` the CUDA-event time of the device fill;
- ``fit_power_law`` follows harness.py:324-345.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from . import engine
from .grid import INPAINT, READABLE


class SpecError(ValueError):
    """An inconsistent synthetic problem (harness.py:20)."""


class DegenerateFitError(ValueError):
    """A power-law fit whose N values do not spread (harness.py:24)."""


@dataclass(frozen=True)
class SyntheticProblem:
    """Two-tone scene on the rectangle ``omega`` with the unknown rectangle
    ``domain`` strictly inside it (harness.py:27-47).  ``geometry`` "line":
    a band of perpendicular half-width ``half_width`` through the centre at
    ``theta_deg``; "step": the two half-planes of that line.  ``colors`` =
    (ink, background), scalars or equal-length channel tuples."""

    omega: tuple = (-1.0, 1.0, -0.5, 0.5)
    domain: tuple = (-0.8, 0.8, -0.3, 0.3)
    geometry: str = "line"
    theta_deg: float = 73.0
    half_width: float = 0.05
    colors: tuple = (0.0, 1.0)
    resolution: tuple = (200, 100)

    def with_resolution(self, resolution) -> "SyntheticProblem":
        return replace(self, resolution=(int(resolution[0]), int(resolution[1])))


@dataclass(frozen=True)
class PowerLawFit:
    """value ~ amplitude * N**alpha; residual = RMS misfit in log-log space."""

    amplitude: float
    alpha: float
    residual: float


def _check(spec: SyntheticProblem) -> None:
    """harness.py:59-76 (same conditions and messages)."""
    ox0, ox1, oy0, oy1 = spec.omega
    dx0, dx1, dy0, dy1 = spec.domain
    if not (ox0 < ox1 and oy0 < oy1):
        raise SpecError("omega rectangle is empty")
    if not (ox0 < dx0 < dx1 < ox1 and oy0 < dy0 < dy1 < oy1):
        raise SpecError("domain must lie strictly inside omega")
    if spec.geometry not in ("line", "step"):
        raise SpecError(f"unknown geometry {spec.geometry!r}")
    if spec.geometry == "line" and not (spec.half_width > 0.0):
        raise SpecError("line half_width must be positive")
    if min(spec.resolution) < 2:
        raise SpecError("resolution must be at least 2x2")
    if len(spec.colors) != 2:
        raise SpecError("colors must give exactly two tones")


def _tones(colors) -> np.ndarray:
    """(2, C) array of the two tones (harness.py:79-84)."""
    ink = np.atleast_1d(np.asarray(colors[0], dtype=np.float64))
    bg = np.atleast_1d(np.asarray(colors[1], dtype=np.float64))
    if ink.ndim != 1 or ink.shape != bg.shape:
        raise SpecError("the two colors must have the same channel count")
    return np.stack([ink, bg])


def pixel_centers(spec: SyntheticProblem):
    """Continuum x (W,) and y (H,) of the pixel centres; row 0 is the top
    (y falls with the row index) -- harness.py:86-97."""
    ox0, ox1, oy0, oy1 = spec.omega
    W, H = spec.resolution
    hx = (ox1 - ox0) / W
    hy = (oy1 - oy0) / H
    return ox0 + (np.arange(W) + 0.5) * hx, oy1 - (np.arange(H) + 0.5) * hy


def _geometry(spec: SyntheticProblem):
    ox0, ox1, oy0, oy1 = spec.omega
    th = math.radians(spec.theta_deg)
    return (ox0 + ox1) / 2.0, (oy0 + oy1) / 2.0, math.sin(th), math.cos(th)


def render_problem(spec: SyntheticProblem):
    """Host rasterisation -> (image (H,W,C) f64, labels (H,W) u8, truth).

    The unknown rectangle is blanked to 0 and labelled Inpaint; the rest is
    Readable (harness.py:100-127)."""
    _check(spec)
    xs, ys = pixel_centers(spec)
    cx, cy, s, c = _geometry(spec)
    X = xs[None, :]
    Y = ys[:, None]
    # signed distance to the centre line, numpy's operation order
    d = (-(X - cx)) * s + (Y - cy) * c
    tones = _tones(spec.colors)
    if spec.geometry == "line":
        which = 1 - (np.abs(d) <= spec.half_width).astype(np.intp)  # 0 = ink band
    else:
        which = (d > 0.0).astype(np.intp)
    truth = tones[which]
    dx0, dx1, dy0, dy1 = spec.domain
    unknown = (X >= dx0) & (X <= dx1) & (Y >= dy0) & (Y <= dy1)
    labels = np.where(unknown, INPAINT, READABLE).astype(np.uint8)
    image = np.where(unknown[..., None], 0.0, truth)
    return image, labels, truth


def render_problem_device(spec: SyntheticProblem, device=None, dtype=None):
    """The same rasterisation written straight into device memory.

    Returns (image (H,W,C), labels (H,W) uint8) CUDA tensors; values equal
    ``render_problem``'s bit for bit in float64 (``dtype`` may narrow the
    image, e.g. torch.float32 for the engine's native layout)."""
    import torch

    _check(spec)
    dev = device or torch.device("cuda")
    f64 = torch.float64
    ox0, ox1, oy0, oy1 = spec.omega
    W, H = spec.resolution
    hx = (ox1 - ox0) / W
    hy = (oy1 - oy0) / H
    xs = ox0 + (torch.arange(W, dtype=f64, device=dev) + 0.5) * hx
    ys = oy1 - (torch.arange(H, dtype=f64, device=dev) + 0.5) * hy
    cx, cy, s, c = _geometry(spec)
    X = xs[None, :]
    Y = ys[:, None]
    d = (-(X - cx)) * s + (Y - cy) * c
    tones = torch.from_numpy(_tones(spec.colors)).to(dev)
    if spec.geometry == "line":
        which = 1 - (d.abs() <= spec.half_width).long()
    else:
        which = (d > 0.0).long()
    del d
    dx0, dx1, dy0, dy1 = spec.domain
    unknown = (X >= dx0) & (X <= dx1) & (Y >= dy0) & (Y <= dy1)
    labels = torch.where(unknown, INPAINT, READABLE).to(torch.uint8)
    image = tones[which]
    image[unknown] = 0.0
    if dtype is not None and dtype != f64:
        image = image.to(dtype)
    return image.contiguous(), labels.contiguous()


def shell_count(spec: SyntheticProblem) -> int:
    """Onion shells of the rendered rectangle, (min(h, w) + 1) // 2
    (harness.py:130-137)."""
    _, labels, _ = render_problem(spec)
    h = int((labels == INPAINT).any(axis=1).sum())
    w = int((labels == INPAINT).any(axis=0).sum())
    return (min(h, w) + 1) // 2


def stripe_family(heights=(50, 70, 100, 140, 200, 280, 400, 500)) -> list:
    """The paper's complexity problem: omega = [0,4]x[0,1], D = [0.4,3.96]x
    [0.2,0.8], one horizontal stripe, resolutions 4h x h (harness.py:261-274).
    Heights up to 5000 reach N = 1e8 px on the GPU."""
    return [SyntheticProblem(omega=(0.0, 4.0, 0.0, 1.0), domain=(0.4, 3.96, 0.2, 0.8),
                             geometry="line", theta_deg=0.0, half_width=0.05,
                             colors=(0.0, 1.0), resolution=(4 * int(h), int(h)))
            for h in heights]


def _default_params():
    from .engine import FillParams

    # smart order off and g identically zero: the study isolates the fill loop
    return FillParams(r=3, mu=50.0, order="onion", neighborhood="rotated_ball",
                      g_source="fixed", g_fixed=(0.0, 0.0))


def scaling_study(problems, params=None, tracked: bool = True, repeats: int = 3,
                  device=None) -> list:
    """Fill every problem on the GPU; one row per problem (harness.py:277-306).

    Row keys as the reference: ``N`` (= W*H), ``seconds`` (here: the best of
    ``repeats`` CUDA-event timings of the device fill, inputs resident),
    ``threads_max`` (widest lane request: the largest frontier when tracked,
    W*H otherwise), ``iterations``, ``work_total`` (tracked only, the
    reference's F*ceil(log2 candidates) sum, tracker.py:127-134); plus
    ``inpaint_px`` = |D_h|, the paper's N."""
    import torch

    from . import _native as N
    from ._device import fill_device
    from .tracker import WorkMetrics

    p = params or _default_params()
    dev = device or N.require_cuda()
    out = []
    for spec in problems:
        img, lab = render_problem_device(spec, dev, torch.float32)
        W, H = spec.resolution
        img = img.reshape(1, H, W, -1)
        lab = lab.reshape(1, H, W)
        res = fill_device(img, lab, None, p, tracked=tracked, rows_cap=min(H * W + 1, 1 << 20))
        ws = res["workspace"]
        best = math.inf
        for _ in range(max(1, repeats)):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            res = fill_device(img, lab, None, p, tracked=tracked, workspace=ws,
                              rows_cap=min(H * W + 1, 1 << 20))
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        stats = res["stats"][0].cpu().numpy()
        iters = int(stats[N.STAT_ITERATIONS])
        frows = res["rows"][0, :iters].cpu().numpy()
        row = {"N": W * H, "seconds": best, "iterations": iters,
               "inpaint_px": int(stats[N.STAT_INPAINT])}
        if tracked:
            wm = WorkMetrics()
            for k in range(iters):
                F = int(frows[k, 0])
                cand = int(frows[k + 1, 0]) if k + 1 < iters else int(stats[N.STAT_LAST_FRONTIER])
                wm.rows.append((k, F, cand, F, int(frows[k, 1])))
            row["threads_max"] = wm.threads_max
            row["work_total"] = wm.work_total
        else:
            row["threads_max"] = W * H
            row["work_total"] = None
        out.append(row)
        del img, lab, res, ws
    return out


def scaling_csv(rows) -> str:
    """harness.py:309-315."""
    body = "".join(f"{r['N']},{r['seconds']:.6g},{r['threads_max']},{r['iterations']}\n"
                   for r in rows)
    return "N,seconds,threads_max,iterations\n" + body


def fit_power_law(points) -> PowerLawFit:
    """Least-squares line through (log N, log value) (harness.py:324-345)."""
    pts = [(float(n), float(v)) for n, v in points]
    if len(pts) < 2:
        raise ValueError("need at least two points")
    if any(n <= 0 or v <= 0 for n, v in pts):
        raise ValueError("points must be positive")
    ln = np.array([math.log(n) for n, _ in pts])
    lv = np.array([math.log(v) for _, v in pts])
    if float(np.ptp(ln)) == 0.0:
        raise DegenerateFitError("all N equal; exponent is undetermined")
    alpha, intercept = np.polyfit(ln, lv, 1)
    miss = lv - (alpha * ln + intercept)
    return PowerLawFit(amplitude=float(math.exp(intercept)), alpha=float(alpha),
                       residual=float(np.sqrt(np.mean(miss * miss))))


def plot_script(csv_name: str, x: str = "N", y: str = "threads_max") -> str:
    """A gnuplot script plotting one study CSV on log-log axes (harness.py:346-352)."""
    return ("set datafile separator ','\n"
            "set logscale xy\n"
            f"plot '{csv_name}' using '{x}':'{y}' with linespoints title '{y}'\n")


# ---------------------------------------------------------------- analysis
# Measurements on filled renderings (harness.py:140-258): host arithmetic on
# the engine's output, the fills themselves run on the device.

def row_profile(u, spec: SyntheticProblem, y_value: float):
    """Channel 0 along the pixel row whose centre is nearest to continuum y
    (harness.py:140-144): (x, profile)."""
    x, y = pixel_centers(spec)
    row = int(np.argmin(np.abs(y - y_value)))
    return x, np.asarray(u[row, :, 0], dtype=np.float64)


def _crossing(x, p, level, start, step):
    """Walk from ``start`` in ``step`` while p < level; interpolate the
    crossing between the last sample below and the first at/above it."""
    k = start
    while p[k] < level:
        k += step
        if k < 0 or k >= p.size:
            return None, None
    a = k - step
    frac = (level - p[a]) / (p[k] - p[a])
    return x[a] + frac * (x[k] - x[a]), k


def rise_width(x, profile, ink: float, bg: float, lo_frac: float = 0.1,
               hi_frac: float = 0.9) -> float:
    """Mean 10-90 transition width of a dark band's two edges, in continuum
    units (harness.py:147-181); inf once the band no longer reaches the low
    level or a crossing runs off the row."""
    p = np.asarray(profile, dtype=np.float64)
    lo, hi = ink + lo_frac * (bg - ink), ink + hi_frac * (bg - ink)
    bottom = int(np.argmin(p))
    if p[bottom] >= lo:
        return math.inf
    widths = []
    for step in (-1, +1):
        x_lo, k_lo = _crossing(x, p, lo, bottom, step)
        if x_lo is None:
            return math.inf
        x_hi, _ = _crossing(x, p, hi, k_lo, step)
        if x_hi is None:
            return math.inf
        widths.append(abs(x_hi - x_lo))
    return 0.5 * (widths[0] + widths[1])


def measure_line_angle(u, labels, spec: SyntheticProblem, margin_rows: int = 2,
                       depth_frac: float = 0.4) -> float:
    """Angle (degrees mod 180) of the dark band the fill extended into the
    unknown rows: per-row darkness centroids over the first depth_frac of
    them (after margin_rows), a least-squares slope dx/dy, converted to a
    continuum angle (harness.py:184-213)."""
    x, y = pixel_centers(spec)
    background = float(np.max(_tones(spec.colors)))
    rows = np.flatnonzero((np.asarray(labels) == INPAINT).any(axis=1))
    last = max(margin_rows + 2, int(math.ceil(depth_frac * rows.size)))
    cx, cy = [], []
    for j in rows[margin_rows:last]:
        dark = np.clip(background - np.asarray(u[j, :, 0], dtype=np.float64), 0.0, None)
        mass = float(dark.sum())
        if mass > 1e-12:
            cx.append(float((dark * x).sum()) / mass)
            cy.append(float(y[j]))
    if len(cx) < 2:
        raise ValueError("no dark band found in the unknown rows")
    slope = float(np.polyfit(cy, cx, 1)[0])
    return math.degrees(math.atan2(1.0, slope)) % 180.0


def _line_guide(spec: SyntheticProblem):
    """Unit guide along the scene's line, image coordinates (rows grow
    downwards): (cos theta, -sin theta) (harness.py:216-219)."""
    th = math.radians(spec.theta_deg)
    return (math.cos(th), -math.sin(th))


def degradation_study(spec: SyntheticProblem, resolutions, cross_sections=(0.3, 0.25, 0.0),
                      params=None) -> list:
    """Band transition widths across depths and scales (harness.py:222-250):
    every rendering is filled on the GPU with a fixed guide along the true
    line and each cross-section's 10-90 width measured."""
    out = []
    for res in resolutions:
        scene = spec.with_resolution(res)
        image, labels, _ = render_problem(scene)
        p = params or engine.FillParams(r=3, mu=50.0, order="smart",
                                        neighborhood="rotated_ball", g_source="fixed",
                                        g_fixed=_line_guide(scene))
        filled, report = engine.inpaint(image, labels, None, p)
        tones = _tones(scene.colors)
        ink, bg = float(np.min(tones)), float(np.max(tones))
        for yv in cross_sections:
            xs, prof = row_profile(filled, scene, float(yv))
            out.append({"resolution": tuple(scene.resolution), "y": float(yv),
                        "width": rise_width(xs, prof, ink, bg),
                        "iterations": report.iterations})
    return out


def degradation_csv(rows) -> str:
    """W,H,y,width rows of a degradation study (harness.py:253-258)."""
    body = "".join(f"{r['resolution'][0]},{r['resolution'][1]},{r['y']:.10g},{r['width']:.10g}\n"
                   for r in rows)
    return "W,H,y,width\n" + body
