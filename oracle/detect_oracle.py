"""CPU oracle for automatic spline detection -- TEST INFRASTRUCTURE ONLY.

A numpy / scipy restatement of the reference's detection pipeline
(/root/reference/pkg/src/guidefill/guide.py:55-283: compute_ring,
detect_edge_seeds, _cluster_seeds, make_spline, detect_splines), the checker
for the device path (paper_1611_05319_b200/csrc/gf_detect.cu,
guide.detect_splines).  Only ``tests/`` import it.

Parity status: UNPINNED for the Canny step.  The reference calls
``skimage.feature.canny`` (guide.py:192; pyproject.toml pins only
scikit-image >= 0.21), which is not installed in this image.  ``canny`` below
restates scikit-image's published algorithm (skimage/feature/_canny.py since
0.19: ``_preprocess`` masked Gaussian with bleed-over, ``ndi.sobel``,
``_nonmaximum_suppression_bilinear``, hysteresis by ``ndi.label``); it is
checked against the reference's own detection tests (test_guide.py:154-216:
seeds {(30, 11), (30, 48)} on the vertical-edge block, a 45 degree spline,
no spline for a grazing edge, none on a constant image), not against
scikit-image outputs.  Everything around Canny (ring, strengths, clustering,
tensor, rays) is the reference code restated with the same numpy / scipy
calls.
"""

from __future__ import annotations

import math

import numpy as np
from scipy import ndimage

from .guidefill_oracle import tensor_field

READABLE, INPAINT = 0, 255
DEFAULT_SIGMA, DEFAULT_RHO, DEFAULT_LAMBDA = 2.0, 4.0, 1e-5
CANNY_LOW, CANNY_HIGH = 0.08, 0.2
SEED_CLUSTER_RADIUS = 3.0


def ring_distance(sigma=DEFAULT_SIGMA, rho=DEFAULT_RHO):  # guide.py:57-59
    return int(math.ceil(2.0 * sigma + 2.0 * rho)) + 1


def cascade_radius(sigma=DEFAULT_SIGMA, rho=DEFAULT_RHO):  # guide.py:62-64
    return int(math.ceil(2.0 * sigma + 2.0 * rho))


def compute_ring(labels, sigma=DEFAULT_SIGMA, rho=DEFAULT_RHO):  # guide.py:65-88
    obstacle = labels != READABLE
    if not obstacle.any():
        raise ValueError("no Inpaint or Bystander pixels to ring")
    dist = ndimage.distance_transform_cdt(~obstacle, metric="chessboard")
    ring = dist == ring_distance(sigma, rho)
    blocked = ndimage.binary_dilation(obstacle, structure=np.ones((3, 3), dtype=bool),
                                      iterations=cascade_radius(sigma, rho))
    ring &= ~blocked
    if not ring.any():
        raise ValueError("empty ring")
    j, i = np.nonzero(ring)
    return set(zip(i.tolist(), j.tolist()))


def _nms_bilinear(isobel, jsobel, magn, eroded_mask, low):
    """skimage _nonmaximum_suppression_bilinear, vectorised: the magnitude at
    local maxima (interpolated neighbours across the gradient), 0 elsewhere."""
    H, W = magn.shape
    out = np.zeros_like(magn)
    cand = eroded_mask & (magn >= low)
    xs, ys = np.nonzero(cand)
    m = magn[xs, ys]
    isob = isobel[xs, ys]
    jsob = jsobel[xs, ys]
    up = isob >= 0
    left = jsob >= 0
    c1 = (up & left) | (~up & ~left)
    c2 = np.abs(isob) >= np.abs(jsob)
    with np.errstate(divide="ignore", invalid="ignore"):
        w = np.where(c2, np.abs(jsob) / np.abs(isob), np.abs(isob) / np.abs(jsob))
    # neighbour offsets per case: (n11, n12, n21, n22) as (dx, dy)
    cases = {
        (True, True): ((1, 0), (1, 1), (-1, 0), (-1, -1)),
        (True, False): ((0, 1), (1, 1), (0, -1), (-1, -1)),
        (False, True): ((1, 0), (1, -1), (-1, 0), (-1, 1)),
        (False, False): ((0, -1), (1, -1), (0, 1), (-1, 1)),
    }
    keep = np.zeros(xs.size, dtype=bool)
    for (a, b), offs in cases.items():
        sel = (c1 == a) & (c2 == b)
        if not sel.any():
            continue
        x, y = xs[sel], ys[sel]
        n11, n12, n21, n22 = (magn[x + dx, y + dy] for dx, dy in offs)
        ws = w[sel]
        keep[sel] = ((n12 * ws + n11 * (1.0 - ws) <= m[sel]) &
                     (n22 * ws + n21 * (1.0 - ws) <= m[sel]))
    out[xs[keep], ys[keep]] = m[keep]
    return out


def canny(image, sigma, low_threshold, high_threshold, mask):
    """skimage.feature.canny(image, sigma, low, high, mask) restated (mode
    'constant', cval 0, absolute thresholds)."""
    image = np.asarray(image, dtype=np.float64)
    mask = np.asarray(mask, dtype=bool)
    kw = dict(sigma=sigma, mode="constant", cval=0.0, truncate=4.0)
    bleed_over = ndimage.gaussian_filter(mask.astype(np.float64), **kw) + np.finfo(np.float64).eps
    masked = np.zeros_like(image)
    masked[mask] = image[mask]
    smoothed = ndimage.gaussian_filter(masked, **kw)
    smoothed /= bleed_over
    eroded = ndimage.binary_erosion(mask, ndimage.generate_binary_structure(2, 2), border_value=0)
    jsobel = ndimage.sobel(smoothed, axis=1)
    isobel = ndimage.sobel(smoothed, axis=0)
    magnitude = isobel * isobel
    magnitude += jsobel * jsobel
    np.sqrt(magnitude, out=magnitude)
    low_masked = _nms_bilinear(isobel, jsobel, magnitude, eroded, low_threshold)
    low_mask = low_masked > 0
    labels, count = ndimage.label(low_mask, np.ones((3, 3), bool))
    if count == 0:
        return low_mask
    high_mask = low_mask & (low_masked >= high_threshold)
    good = np.zeros(count + 1, dtype=bool)
    good[np.unique(labels[high_mask])] = True
    good[0] = False
    return good[labels]


def _smooth(arr, s):  # guide.py:46-48
    return ndimage.gaussian_filter(arr, sigma=s, truncate=2.0, mode="constant", cval=0.0)


def _gray(image):  # guide.py:51-52
    return image.mean(axis=2) if image.ndim == 3 else image


def detect_hits(image, labels, sigma=DEFAULT_SIGMA, rho=DEFAULT_RHO, low=CANNY_LOW,
                high=CANNY_HIGH):
    """guide.py:183-196 before the clustering: (i, j, strength) in (j, i) order."""
    ring = compute_ring(labels, sigma, rho)
    obstacle = labels != READABLE
    dist = ndimage.distance_transform_cdt(~obstacle, metric="chessboard")
    d_ring = ring_distance(sigma, rho)
    half = int(math.ceil(2.0 * sigma)) + 1
    annulus = (dist >= d_ring - half) & (dist <= d_ring + half) & (labels == READABLE)
    gray = _gray(image)
    edges = canny(gray, sigma, low, high, annulus)
    gy, gx = np.gradient(_smooth(gray, sigma))
    strength = np.hypot(gx, gy)
    return [(i, j, float(strength[j, i])) for (i, j) in sorted(ring, key=lambda p: (p[1], p[0]))
            if edges[j, i]]


def cluster_seeds(hits, radius=SEED_CLUSTER_RADIUS):  # guide.py:200-207
    kept = []
    for i, j, s in sorted(hits, key=lambda h: (-h[2], h[1], h[0])):
        if all((i - ki) ** 2 + (j - kj) ** 2 > radius * radius for ki, kj, _ in kept):
            kept.append((i, j, s))
    kept.sort(key=lambda h: (h[1], h[0]))
    return kept


def detect_edge_seeds(image, labels, sigma=DEFAULT_SIGMA, rho=DEFAULT_RHO, low=CANNY_LOW,
                      high=CANNY_HIGH):  # guide.py:177-197
    return cluster_seeds(detect_hits(image, labels, sigma, rho, low, high))


def eigen_2x2(a, b, c):  # guide.py:123-136
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    mean = (a + c) / 2.0
    disc = np.sqrt(((a - c) / 2.0) ** 2 + b * b)
    phi_major = 0.5 * np.arctan2(2.0 * b, a - c)
    return mean - disc, mean + disc, -np.sin(phi_major), np.cos(phi_major)


def structure_tensor(image, point, sigma=DEFAULT_SIGMA, rho=DEFAULT_RHO):  # guide.py:139-156
    i, j = int(point[0]), int(point[1])
    ones = np.ones(image.shape[:2])
    J11, J12, J22, _ = tensor_field(image, ones, sigma, rho)
    return np.array([[J11[j, i], J12[j, i]], [J12[j, i], J22[j, i]]])


def make_spline(seed, image, labels, sigma=DEFAULT_SIGMA, rho=DEFAULT_RHO, lam=DEFAULT_LAMBDA):
    """guide.py:210-267: (start, end, direction) or None."""
    i, j = int(seed[0]), int(seed[1])
    J = structure_tensor(image, (i, j), sigma, rho)
    lo, hi, vx, vy = eigen_2x2(J[0, 0], J[0, 1], J[1, 1])
    coherence = math.tanh((float(hi) - float(lo)) / lam)
    H, W = labels.shape
    budget = 2 * ring_distance(sigma, rho)
    step = 0.5
    start = np.array([float(i), float(j)])

    def first_entry(direction):
        for t in np.arange(step, budget + step / 2, step):
            p = start + t * direction
            ii, jj = int(round(p[0])), int(round(p[1]))
            if not (0 <= ii < W and 0 <= jj < H):
                return None
            if labels[jj, ii] == INPAINT:
                return t
        return None

    v = np.array([float(vx), float(vy)])
    t_plus = first_entry(v)
    t_minus = first_entry(-v)
    if t_plus is None and t_minus is None:
        return None
    if t_minus is None or (t_plus is not None and t_plus <= t_minus):
        direction, t_entry = v, t_plus
    else:
        direction, t_entry = -v, t_minus
    t_end = t_entry
    t = t_entry
    limit = 2.0 * (H + W)
    while t < limit:
        t += step
        p = start + t * direction
        ii, jj = int(round(p[0])), int(round(p[1]))
        if not (0 <= ii < W and 0 <= jj < H) or labels[jj, ii] == READABLE:
            break
        t_end = t
    end = start + t_end * direction
    return start, end, (coherence * direction[0], coherence * direction[1])


def detect_splines(image, labels, sigma=DEFAULT_SIGMA, rho=DEFAULT_RHO, lam=DEFAULT_LAMBDA,
                   low=CANNY_LOW, high=CANNY_HIGH):  # guide.py:270-283
    out = []
    for i, j, _ in detect_edge_seeds(image, labels, sigma, rho, low, high):
        sp = make_spline((i, j), image, labels, sigma, rho, lam)
        if sp is not None:
            out.append(sp)
    return out
