"""Seeded synthetic disocclusion scenes for the benchmark configurations.

Restates the generators of SURVEY.md section 8(d) / Appendix C (these are
the survey's own probe recipes, not reference code):

* C1: 512x512 random RGB, one vertical 8 px Inpaint band, one straight
  spline at 30 degrees, r=3, mu=100, smart order.
* C2/C3: 1920x1080 "object-edge disocclusion" frame: a 10x6 grid of
  foreground ellipses (Bystander), the 10 px strip left of each ellipse is
  Inpaint, 6 cubic Bezier guide splines; r=3 (C2) or r=5 (C3), mu=50.
* C4: 3840x2160, 40 px bands, r=4, straight two-point splines standing in
  for the auto-detected ones (the reference detector needs scikit-image,
  which is absent; the spline list is generated once and shared by both
  engines, as BASELINE.md section 3 prescribes).
* C5: 256 C2 frames, per-frame seed 1611 + 7919 f, objects drifting 3 px/frame.

Values do not affect the fill order for the guide-field g source
(SURVEY.md section 0.4), so only the label geometry has to be realistic.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

READABLE = 0
BYSTANDER = 128
INPAINT = 255


@dataclass
class Scene:
    name: str
    image: np.ndarray          # (H, W, 3) float64 in [0, 1]
    labels: np.ndarray         # (H, W) uint8
    splines: list              # list of dicts: points (P,2), kind, direction
    params: dict = field(default_factory=dict)

    @property
    def n_inpaint(self) -> int:
        return int((self.labels == INPAINT).sum())


def _texture(H, W, rng):
    jj, ii = np.mgrid[0:H, 0:W].astype(np.float64)
    img = np.empty((H, W, 3))
    phases = rng.uniform(0.0, 2.0 * math.pi, 3)
    stripes = 0.08 * np.sign(np.sin((0.8 * ii + 0.6 * jj) / 11.0))
    for c in range(3):
        img[..., c] = 0.5 + 0.35 * np.sin(ii / (90.0 + 40.0 * c) + jj / (140.0 + 30.0 * c) + phases[c])
    img += stripes[..., None]
    img += rng.uniform(0.0, 0.05, size=img.shape)
    np.clip(img, 0.0, 1.0, out=img)
    return img


def disocclusion_frame(H=1080, W=1920, band=10, gx=10, gy=6, n_spl=6, seed=1611, frame=0,
                       spline_kind="bezier"):
    """Object-edge disocclusion frame."""
    rng = np.random.default_rng(seed + 7919 * frame)
    cw = W / gx
    ch = H / gy
    ellipses = []
    for cy_i in range(gy):
        for cx_i in range(gx):
            cx = (cx_i + 0.5) * cw + rng.uniform(-0.1, 0.1) * cw + 3.0 * frame
            cy = (cy_i + 0.5) * ch + rng.uniform(-0.1, 0.1) * ch
            rx = rng.uniform(0.22, 0.32) * cw
            ry = rng.uniform(0.30, 0.42) * ch
            ellipses.append((cx, cy, rx, ry))
    obj = np.zeros((H, W), dtype=bool)
    for cx, cy, rx, ry in ellipses:
        j0 = max(0, int(math.floor(cy - ry)) - 1)
        j1 = min(H, int(math.ceil(cy + ry)) + 2)
        i0 = max(0, int(math.floor(cx - rx)) - 1)
        i1 = min(W, int(math.ceil(cx + rx)) + 2)
        if j0 >= j1 or i0 >= i1:
            continue
        jj, ii = np.mgrid[j0:j1, i0:i1].astype(np.float64)
        obj[j0:j1, i0:i1] |= ((ii - cx) / rx) ** 2 + ((jj - cy) / ry) ** 2 <= 1.0
    hole = np.zeros((H, W), dtype=bool)
    for s in range(1, band + 1):
        hole[:, :W - s] |= obj[:, s:]
    hole &= ~obj
    labels = np.full((H, W), READABLE, dtype=np.uint8)
    labels[obj] = BYSTANDER
    labels[hole] = INPAINT
    image = _texture(H, W, rng)
    image[hole] = 0.0

    splines = []
    picks = rng.choice(len(ellipses), size=n_spl, replace=False)
    L = 3.0 * band + 30.0
    for k, e in enumerate(picks):
        cx, cy, rx, ry = ellipses[int(e)]
        x_edge = cx - rx
        y0 = cy + rng.uniform(-0.5, 0.5) * ry
        a = rng.uniform(-0.6, 0.6)
        p0 = np.array([x_edge - L, y0 - L * math.tan(a)])
        p3 = np.array([x_edge + 2.0, y0])
        d = p3 - p0
        unit = d / math.hypot(d[0], d[1])
        if spline_kind == "bezier":
            p1 = p0 + d / 3.0 + np.array([0.0, rng.uniform(-8.0, 8.0)])
            p2 = p0 + 2.0 * d / 3.0 + np.array([0.0, rng.uniform(-8.0, 8.0)])
            pts = np.stack([p0, p1, p2, p3])
            direction = (0.97 * unit[0], 0.97 * unit[1])
        else:
            pts = np.stack([p0, p3 + 2.0 * unit * band])
            direction = (float(np.tanh(4.0)) * unit[0], float(np.tanh(4.0)) * unit[1])
        splines.append(dict(id=f"s{k}", points=pts, kind=spline_kind,
                            direction=(float(direction[0]), float(direction[1]))))
    return image, labels, splines


def config(name: str, frame: int = 0) -> Scene:
    """Build one of the BASELINE.json configurations (C1..C5 frame f)."""
    name = name.upper()
    if name == "C1":
        rng = np.random.default_rng(1611)
        H = W = 512
        image = rng.random((H, W, 3))
        labels = np.full((H, W), READABLE, dtype=np.uint8)
        labels[:, 252:260] = INPAINT
        image[labels == INPAINT] = 0.0
        th = math.radians(30.0)
        c = np.array([255.5, 255.5])
        u = np.array([math.cos(th), math.sin(th)])
        pts = np.stack([c - 300.0 * u, c + 300.0 * u])
        spl = [dict(id="s0", points=pts, kind="polyline",
                    direction=(0.98 * u[0], 0.98 * u[1]))]
        return Scene("C1", image, labels, spl,
                     dict(r=3, mu=100.0, order="smart", neighborhood="rotated_ball"))
    if name in ("C2", "C3", "C5"):
        image, labels, spl = disocclusion_frame(frame=frame if name == "C5" else 0)
        r = 5 if name == "C3" else 3
        return Scene(name, image, labels, spl,
                     dict(r=r, mu=50.0, order="smart", neighborhood="rotated_ball"))
    if name == "C4":
        image, labels, spl = disocclusion_frame(H=2160, W=3840, band=40, spline_kind="polyline")
        return Scene("C4", image, labels, spl,
                     dict(r=4, mu=50.0, order="smart", neighborhood="rotated_ball"))
    raise ValueError(f"unknown config {name!r}")


def small_scene(H, W, band, gx, gy, n_spl, seed, frame=0, spline_kind="bezier"):
    """Scaled-down disocclusion frame for fast parity tests."""
    image, labels, spl = disocclusion_frame(H=H, W=W, band=band, gx=gx, gy=gy, n_spl=n_spl,
                                            seed=seed, frame=frame, spline_kind=spline_kind)
    return Scene(f"small{H}x{W}", image, labels, spl,
                 dict(r=3, mu=50.0, order="smart", neighborhood="rotated_ball"))


def _frame_geometry(H, W, band, gx, gy, n_spl, seed, frame, spline_kind="bezier"):
    """The random draws of ``disocclusion_frame`` in its RNG order, without
    materialising the texture: ellipses, texture phases, (skip the H*W*3 noise
    draws), splines.  Returns (ellipses, phases, splines)."""
    rng = np.random.default_rng(seed + 7919 * frame)
    cw = W / gx
    ch = H / gy
    ellipses = []
    for cy_i in range(gy):
        for cx_i in range(gx):
            cx = (cx_i + 0.5) * cw + rng.uniform(-0.1, 0.1) * cw + 3.0 * frame
            cy = (cy_i + 0.5) * ch + rng.uniform(-0.1, 0.1) * ch
            rx = rng.uniform(0.22, 0.32) * cw
            ry = rng.uniform(0.30, 0.42) * ch
            ellipses.append((cx, cy, rx, ry))
    phases = rng.uniform(0.0, 2.0 * math.pi, 3)
    rng.bit_generator.advance(H * W * 3)  # the noise: one 64-bit draw per double
    splines = []
    picks = rng.choice(len(ellipses), size=n_spl, replace=False)
    L = 3.0 * band + 30.0
    for k, e in enumerate(picks):
        cx, cy, rx, ry = ellipses[int(e)]
        x_edge = cx - rx
        y0 = cy + rng.uniform(-0.5, 0.5) * ry
        a = rng.uniform(-0.6, 0.6)
        p0 = np.array([x_edge - L, y0 - L * math.tan(a)])
        p3 = np.array([x_edge + 2.0, y0])
        d = p3 - p0
        unit = d / math.hypot(d[0], d[1])
        if spline_kind == "bezier":
            p1 = p0 + d / 3.0 + np.array([0.0, rng.uniform(-8.0, 8.0)])
            p2 = p0 + 2.0 * d / 3.0 + np.array([0.0, rng.uniform(-8.0, 8.0)])
            pts = np.stack([p0, p1, p2, p3])
            direction = (0.97 * unit[0], 0.97 * unit[1])
        else:
            pts = np.stack([p0, p3 + 2.0 * unit * band])
            direction = (float(np.tanh(4.0)) * unit[0], float(np.tanh(4.0)) * unit[1])
        splines.append(dict(id=f"s{k}", points=pts, kind=spline_kind,
                            direction=(float(direction[0]), float(direction[1]))))
    return ellipses, phases, splines


def video_batch_device(frames, device, H=1080, W=1920, band=10, gx=10, gy=6, n_spl=6, seed=1611,
                       dtype=None):
    """C5 video frames rendered straight into HBM (SURVEY.md section 8(d):
    "generated on device").

    Returns (images (N, H, W, 3), labels (N, H, W) uint8, splines per frame).
    Labels and splines are bit-identical to ``disocclusion_frame(frame=f)``
    (same RNG draws; the ellipse test is the same sequence of IEEE double
    operations), so the fill order and |D| equal the host generator's.  The
    texture is the same formula evaluated on the GPU with device noise: its
    values differ from the host frame's, which changes only output colours
    (SURVEY.md section 0.4), not the work.
    """
    import torch

    dtype = dtype or torch.float32
    frames = list(frames)
    n = len(frames)
    images = torch.empty((n, H, W, 3), dtype=dtype, device=device)
    labels = torch.empty((n, H, W), dtype=torch.uint8, device=device)
    jj = torch.arange(H, dtype=torch.float64, device=device).view(H, 1)
    ii = torch.arange(W, dtype=torch.float64, device=device).view(1, W)
    stripes = 0.08 * torch.sign(torch.sin((0.8 * ii + 0.6 * jj) / 11.0))
    gen = torch.Generator(device=device)
    spl_all = []
    for b, f in enumerate(frames):
        ellipses, phases, spl = _frame_geometry(H, W, band, gx, gy, n_spl, seed, f)
        spl_all.append(spl)
        obj = torch.zeros((H, W), dtype=torch.bool, device=device)
        for cx, cy, rx, ry in ellipses:
            j0 = max(0, int(math.floor(cy - ry)) - 1)
            j1 = min(H, int(math.ceil(cy + ry)) + 2)
            i0 = max(0, int(math.floor(cx - rx)) - 1)
            i1 = min(W, int(math.ceil(cx + rx)) + 2)
            if j0 >= j1 or i0 >= i1:
                continue
            a = (ii[:, i0:i1] - cx) / rx
            c = (jj[j0:j1] - cy) / ry
            obj[j0:j1, i0:i1] |= (a * a + c * c) <= 1.0
        hole = torch.zeros_like(obj)
        for s in range(1, band + 1):
            hole[:, :W - s] |= obj[:, s:]
        hole &= ~obj
        lab = labels[b]
        lab.fill_(READABLE)
        lab.masked_fill_(obj, BYSTANDER)
        lab.masked_fill_(hole, INPAINT)
        gen.manual_seed(seed + 7919 * f)
        img = torch.empty((H, W, 3), dtype=torch.float64, device=device)
        for ch in range(3):
            img[..., ch] = 0.5 + 0.35 * torch.sin(ii / (90.0 + 40.0 * ch) + jj / (140.0 + 30.0 * ch)
                                                 + float(phases[ch]))
        img += stripes[..., None]
        img += torch.rand((H, W, 3), generator=gen, dtype=torch.float64, device=device) * 0.05
        img.clamp_(0.0, 1.0)
        img[hole] = 0.0
        images[b].copy_(img)
    return images, labels, spl_all
