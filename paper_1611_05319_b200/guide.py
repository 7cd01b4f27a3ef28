"""Guide field from splines -- drop-in for the reference's build_guide_field.

``build_guide_field`` (guide.py:303-327) runs the GPU rasteriser
(gf_guide_field): per Inpaint pixel, the minimum distance to each spline's
flattened polyline, the first nearest spline, and the Gaussian falloff
g = dir * exp(-d^2 / (2 eta^2)), zero beyond 3 eta and outside D.

``coherence_directions`` (guide.py:330-355) runs the masked structure tensor
on the device (gf_coherence_directions).

Automatic spline detection (guide.py:55-283) runs on
the device too: ``gf_detect_edges`` computes the measurement ring, Canny on
the annulus (scikit-image's algorithm restated -- scikit-image is absent from
this image, so that step's parity rests on the reference's own detection
tests) and the seed strengths; ``gf_structure_eigen`` the plain structure
tensor at the seeds; ``gf_trace_rays`` make_spline's entry search and
extension.  Only the seed clustering of a handful of hits (guide.py:200-207)
and the Spline records are host work, as in the reference.
"""

from __future__ import annotations

import math

import numpy as np

from .grid import INPAINT, READABLE
from .splines import Spline

DEFAULT_SIGMA = 2.0
DEFAULT_RHO = 4.0
DEFAULT_LAMBDA = 1e-5
DEFAULT_ETA = 3.0
CANNY_LOW = 0.08
CANNY_HIGH = 0.2
SEED_CLUSTER_RADIUS = 3.0


class EmptyRingError(ValueError):
    """No pixel is far enough from the unknown region to measure on."""


class WindowOverlapError(ValueError):
    """A convolution window reaches into non-Readable territory."""


class ZeroMassError(ValueError):
    """The masked tensor has no readable mass at the queried pixel."""


def ring_distance(sigma: float = DEFAULT_SIGMA, rho: float = DEFAULT_RHO) -> int:
    """Chebyshev clearance of the measurement ring (guide.py:57-59)."""
    import math

    return int(math.ceil(2.0 * sigma + 2.0 * rho)) + 1


def cascade_radius(sigma: float = DEFAULT_SIGMA, rho: float = DEFAULT_RHO) -> int:
    """Chebyshev radius of the smoothing-window cascade (guide.py:62-64)."""
    import math

    return int(math.ceil(2.0 * sigma + 2.0 * rho))


def _image3(image):
    img = np.asarray(image, dtype=np.float64)
    return img[:, :, None] if img.ndim == 2 else img


def _detect_device(image, labels, sigma, rho, low, high, want_ring=False, cap=1 << 16):
    """gf_detect_edges on the device: (hit flat indices, strengths, ring mask)."""
    import ctypes

    import torch
    from . import _native as N

    dev = N.require_cuda()
    lib = N.load()
    img = _image3(image)
    labels = np.ascontiguousarray(labels, dtype=np.uint8)
    H, W, C = img.shape
    d_img = torch.from_numpy(np.ascontiguousarray(img)).to(dev)
    d_lab = torch.from_numpy(labels).to(dev)
    need = lib.gf_detect_workspace_bytes(H, W)
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    idx = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
    strength = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
    ring = torch.empty((H, W), dtype=torch.uint8, device=dev) if want_ring else None
    n = ctypes.c_int32(0)
    N.check(lib.gf_detect_edges(H, W, C, N.ptr(d_img), N.ptr(d_lab), float(sigma), float(rho),
                                float(low), float(high), cap, N.ptr(idx), N.ptr(strength),
                                ctypes.byref(n), N.ptr(ring), None, N.ptr(ws), need,
                                N.stream_ptr()))
    if n.value > cap:
        return _detect_device(image, labels, sigma, rho, low, high, want_ring, n.value)
    k = n.value
    return (idx[:k].cpu().numpy(), strength[:k].cpu().numpy(),
            None if ring is None else ring.cpu().numpy().astype(bool))


def compute_ring(labels, sigma: float = DEFAULT_SIGMA, rho: float = DEFAULT_RHO):
    """Readable pixels at exactly the clearance distance from D u B, as a set
    of (i, j) (guide.py:65-88), computed on the device."""
    labels = np.asarray(labels)
    if not (labels != READABLE).any():
        raise EmptyRingError("no Inpaint or Bystander pixels to ring")
    img = np.zeros(labels.shape + (1,))
    _, _, ring = _detect_device(img, labels, sigma, rho, CANNY_LOW, CANNY_HIGH, want_ring=True,
                                cap=0)
    if not ring.any():
        raise EmptyRingError(
            f"no readable pixel sits {ring_distance(sigma, rho)} px clear of the unknown region")
    j, i = np.nonzero(ring)
    return set(zip(i.tolist(), j.tolist()))


def _cluster_seeds(hits, radius: float = SEED_CLUSTER_RADIUS):
    """Greedy strongest-first suppression of seeds closer than ``radius``
    (guide.py:200-207)."""
    kept = []
    for i, j, s in sorted(hits, key=lambda h: (-h[2], h[1], h[0])):
        if all((i - ki) ** 2 + (j - kj) ** 2 > radius * radius for ki, kj, _ in kept):
            kept.append((i, j, s))
    kept.sort(key=lambda h: (h[1], h[0]))
    return kept


def detect_edge_seeds(image, labels, sigma: float = DEFAULT_SIGMA, rho: float = DEFAULT_RHO,
                      low: float = CANNY_LOW, high: float = CANNY_HIGH):
    """Edge crossings of the measurement ring: [(i, j, strength)]
    (guide.py:177-197).  Ring, Canny and strengths on the device."""
    labels = np.asarray(labels)
    if not (labels != READABLE).any():
        raise EmptyRingError("no Inpaint or Bystander pixels to ring")
    idx, strength, ring = _detect_device(image, labels, sigma, rho, low, high, want_ring=True)
    if not ring.any():
        raise EmptyRingError(
            f"no readable pixel sits {ring_distance(sigma, rho)} px clear of the unknown region")
    W = labels.shape[1]
    order = np.argsort(idx, kind="stable")  # (j, i) order, as the reference sorts the ring
    hits = [(int(p % W), int(p // W), float(s)) for p, s in zip(idx[order], strength[order])]
    return _cluster_seeds(hits)


def eigen_2x2(a, b, c):
    """Eigen split of symmetric [[a, b], [b, c]] (guide.py:123-136): (lambda-,
    lambda+, minor eigenvector x, y)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    mean = (a + c) / 2.0
    disc = np.sqrt(((a - c) / 2.0) ** 2 + b * b)
    phi_major = 0.5 * np.arctan2(2.0 * b, a - c)
    return mean - disc, mean + disc, -np.sin(phi_major), np.cos(phi_major)


def tensor_orientation(J) -> float:
    """Isophote angle of a tensor, minor eigenvector angle mod pi (guide.py:170-174)."""
    import math

    _, _, vx, vy = eigen_2x2(J[0, 0], J[0, 1], J[1, 1])
    return float(np.mod(math.atan2(float(vy), float(vx)), math.pi))


def _eigen_device(image, readable, points, sigma, rho, lam):
    """gf_structure_eigen at (i, j) points: (n, 8) float64 host array."""
    import torch
    from . import _native as N

    dev = N.require_cuda()
    lib = N.load()
    img = _image3(image)
    H, W, C = img.shape
    lab = np.where(np.asarray(readable, dtype=bool), 0, INPAINT).astype(np.uint8)
    pts = np.asarray(points, dtype=np.int64).reshape(-1, 2)
    idx = torch.from_numpy(pts[:, 1] * W + pts[:, 0]).to(dev)
    n = int(idx.numel())
    eig = torch.empty((max(n, 1), 8), dtype=torch.float64, device=dev)
    need = lib.gf_coherence_workspace_bytes(H, W, C)
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    # device copies held in locals: a temporary's memory could be handed to
    # the next allocation before the kernel runs
    d_img = torch.from_numpy(np.ascontiguousarray(img)).to(dev)
    d_lab = torch.from_numpy(lab).to(dev)
    N.check(lib.gf_structure_eigen(H, W, C, N.ptr(d_img), N.ptr(d_lab), n, N.ptr(idx),
                                   float(sigma), float(rho), float(lam), N.ptr(eig), N.ptr(ws),
                                   need, N.stream_ptr()))
    return eig[:n].cpu().numpy()


def _tensor_field(image, indicator, sigma: float, rho: float):
    """Indicator-weighted structure tensor field (guide.py:91-120) on the
    device: (J11, J12, J22, rho mass) planes, every pixel queried.  The
    indicator must be 0 / 1 (all ones: the plain tensor; the Readable mask:
    the masked one)."""
    ind = np.asarray(indicator, dtype=np.float64)
    if not np.all((ind == 0.0) | (ind == 1.0)):
        raise NotImplementedError("the device tensor takes a 0 / 1 indicator")
    img = _image3(image)
    H, W = ind.shape
    jj, ii = np.mgrid[0:H, 0:W]
    e = _eigen_device(img, ind == 1.0, np.stack([ii.ravel(), jj.ravel()], axis=1), sigma, rho,
                      DEFAULT_LAMBDA)
    return tuple(e[:, c].reshape(H, W).copy() for c in (3, 4, 5, 6))


def structure_tensor(image, point, sigma: float = DEFAULT_SIGMA, rho: float = DEFAULT_RHO,
                     labels=None):
    """Smoothed gradient outer-product tensor at one pixel (guide.py:139-156)."""
    i, j = int(point[0]), int(point[1])
    img = _image3(image)
    if labels is not None:
        w = cascade_radius(sigma, rho)
        window = np.asarray(labels)[max(0, j - w):j + w + 1, max(0, i - w):i + w + 1]
        if (window != READABLE).any():
            raise WindowOverlapError(
                f"window of radius {w} around ({i}, {j}) touches non-Readable pixels")
    e = _eigen_device(img, np.ones(img.shape[:2], dtype=bool), [(i, j)], sigma, rho,
                      DEFAULT_LAMBDA)[0]
    return np.array([[e[3], e[4]], [e[4], e[5]]])


def modified_structure_tensor(image, labels, point, sigma: float = DEFAULT_SIGMA,
                              rho: float = DEFAULT_RHO):
    """Masked tensor, usable next to the unknown region (guide.py:159-167)."""
    i, j = int(point[0]), int(point[1])
    e = _eigen_device(image, np.asarray(labels) == READABLE, [(i, j)], sigma, rho,
                      DEFAULT_LAMBDA)[0]
    if e[6] <= 0.0:
        raise ZeroMassError(f"no readable mass within the window at ({i}, {j})")
    return np.array([[e[3], e[4]], [e[4], e[5]]])


def _trace_device(labels, seeds, v, budget):
    """gf_trace_rays: (n, 3) (sign, t_entry, t_end)."""
    import torch
    from . import _native as N

    dev = N.require_cuda()
    lib = N.load()
    labels = np.ascontiguousarray(labels, dtype=np.uint8)
    H, W = labels.shape
    n = len(seeds)
    out = torch.empty((max(n, 1), 3), dtype=torch.float64, device=dev)
    d_lab = torch.from_numpy(labels).to(dev)
    d_seeds = torch.from_numpy(np.ascontiguousarray(seeds, dtype=np.float64).reshape(-1, 2)).to(dev)
    d_v = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64).reshape(-1, 2)).to(dev)
    N.check(lib.gf_trace_rays(H, W, N.ptr(d_lab), n, N.ptr(d_seeds), N.ptr(d_v), float(budget),
                              N.ptr(out), N.stream_ptr()))
    return out[:n].cpu().numpy()


def _splines_from_seeds(seeds, image, labels, sigma, rho, lam, ids):
    labels = np.asarray(labels)
    if not len(seeds):
        return []
    pts = [(int(s[0]), int(s[1])) for s in seeds]
    img = _image3(image)
    eig = _eigen_device(img, np.ones(img.shape[:2], dtype=bool), pts, sigma, rho, lam)
    rays = _trace_device(labels, [(float(i), float(j)) for i, j in pts], eig[:, :2],
                         2 * ring_distance(sigma, rho))
    out = []
    for k, (i, j) in enumerate(pts):
        sign, _, t_end = rays[k]
        if sign == 0.0:
            continue  # no entry within the budget: a grazing edge (guide.py:240-241)
        v = np.array([float(eig[k, 0]), float(eig[k, 1])])
        direction = v if sign > 0 else -v
        start = np.array([float(i), float(j)])
        end = start + t_end * direction
        # make_spline's coherence is Python's math.tanh of the eigenvalue gap
        # (guide.py:224-225), not numpy's: the gap from the device's tensor
        # (a, b, c) with eigen_2x2's numpy ops, then glibc tanh on the host
        a, b, c = float(eig[k, 3]), float(eig[k, 4]), float(eig[k, 5])
        lo, hi = eigen_2x2(a, b, c)[:2]
        coherence = math.tanh((float(hi) - float(lo)) / lam)
        out.append(Spline(id=ids(k), source="auto",
                          direction=(coherence * direction[0], coherence * direction[1]),
                          points=np.stack([start, end])))
    return out


def make_spline(seed, image, labels, sigma: float = DEFAULT_SIGMA, rho: float = DEFAULT_RHO,
                lam: float = DEFAULT_LAMBDA, spline_id: str = "auto-0"):
    """Trace a straight guide spline through a ring seed (guide.py:210-267);
    None when the ray never enters the unknown region."""
    got = _splines_from_seeds([seed], image, labels, sigma, rho, lam, lambda k: spline_id)
    return got[0] if got else None


def detect_splines(image, labels, sigma: float = DEFAULT_SIGMA, rho: float = DEFAULT_RHO,
                   lam: float = DEFAULT_LAMBDA, low: float = CANNY_LOW,
                   high: float = CANNY_HIGH):
    """Full pipeline (guide.py:270-283): ring, seeds, one traced spline per
    surviving seed, ids auto-0, auto-1, ..."""
    seeds = detect_edge_seeds(image, labels, sigma, rho, low, high)
    out = _splines_from_seeds([(i, j) for i, j, _ in seeds], image, labels, sigma, rho, lam,
                              lambda k: f"auto-{k}")
    for k, sp in enumerate(out):
        sp.id = f"auto-{k}"
    return out


def build_guide_field(splines, labels, eta: float = DEFAULT_ETA) -> np.ndarray:
    """(H, W, 2) float64 guide field; exactly zero outside D and beyond 3 eta."""
    import torch
    from . import _native as N
    from ._device import SegmentSet, guide_field_device

    labels = np.asarray(labels)
    H, W = labels.shape
    splines = list(splines)
    if not splines or not (labels == INPAINT).any():
        return np.zeros((H, W, 2))
    from . import _staging

    dev = N.require_cuda()
    segs = SegmentSet.cached(splines, dev)
    d_lab = _staging.upload(np.ascontiguousarray(labels, dtype=np.uint8), dev, "lab")
    return _staging.download(guide_field_device(d_lab, segs, eta))


def coherence_directions(image, readable, ix, iy, sigma: float = DEFAULT_SIGMA,
                         rho: float = DEFAULT_RHO, lam: float = DEFAULT_LAMBDA) -> np.ndarray:
    """Masked-tensor transport directions at the queried pixels: (F, 2) float64
    (guide.py:330-355); 0 where the rho window holds no readable mass."""
    import torch
    from . import _native as N
    from .coherence import coherence_directions_device

    dev = N.require_cuda()
    readable = np.asarray(readable, dtype=bool)
    H, W = readable.shape
    img = np.asarray(image, dtype=np.float64)
    if img.ndim == 2:
        img = img[:, :, None]
    idx = np.asarray(iy, dtype=np.int64) * W + np.asarray(ix, dtype=np.int64)
    if idx.size == 0:
        return np.zeros((0, 2))
    lab = np.where(readable, 0, INPAINT).astype(np.uint8)
    g = coherence_directions_device(torch.from_numpy(np.ascontiguousarray(img)).to(dev),
                                    torch.from_numpy(lab).to(dev),
                                    torch.from_numpy(idx.reshape(-1)).to(dev), sigma, rho, lam)
    return g.cpu().numpy()
