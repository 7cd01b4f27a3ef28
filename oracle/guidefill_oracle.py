"""CPU oracle for the Guidefill fill path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm
(/root/reference/pkg/src/guidefill, arXiv 1611.05319 Algorithm 1) used as the
parity checker for the CUDA engine in ``paper_1611_05319_b200``.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may
import it.  The product path never calls it.

Parity status: PINNED.  ``tests/golden/make_golden.py`` runs the reference
package itself (imported from /root/reference with a ``skimage`` stub) and
stores its outputs as fixtures; ``tests/test_oracle_golden.py`` checks this
restatement against them bit for bit (image bytes, report rows, per-shell
frontier/fill sets, guide fields).

Every floating-point expression keeps the reference's numpy evaluation order
(same ufuncs, same operand order, no fused multiply-add), so the results are
bit-identical to the reference on the same host.  Citations are
``file:line`` under /root/reference/pkg/src/guidefill/.

Extra outputs beyond the reference return values (used by the parity tests):

* ``enter``: per pixel, the shell index at which it joined the frontier
  (-1 if never);
* ``fillshell``: per pixel, the shell index in which it was filled
  (-1 if never, -2 if painted by the unfillable fallback).

Because a frontier pixel stays in the frontier until it is filled, the pair
(enter, fillshell) encodes the full per-shell frontier sets and fill masks:
frontier(k) = {p : enter[p] <= k <= fillshell[p]}, filled(k) = {p : fillshell[p] == k}.
"""

from __future__ import annotations

import math

import numpy as np
from scipy import ndimage

READABLE = 0
BYSTANDER = 128
INPAINT = 255

# (di, dj) order of grid.py:29-33
NEIGHBOR_OFFSETS = (
    (-1, -1), (0, -1), (1, -1),
    (-1, 0), (1, 0),
    (-1, 1), (0, 1), (1, 1),
)


# ----------------------------------------------------------------- lattice

def disk_offsets(r: int) -> np.ndarray:
    """Integer (n, m) with n^2+m^2 <= r^2, meshgrid scan order, centre first.

    grid.py:109-124.  Row k of the result is ball sample k; the engine drops
    row 0 (the centre), engine.py:172.
    """
    span = np.arange(-r, r + 1)
    n_grid, m_grid = np.meshgrid(span, span)
    inside = n_grid * n_grid + m_grid * m_grid <= r * r
    pts = np.stack([n_grid[inside], m_grid[inside]], axis=1).astype(np.float64)
    c = int(np.flatnonzero((pts[:, 0] == 0) & (pts[:, 1] == 0))[0])
    perm = [c] + [k for k in range(len(pts)) if k != c]
    return pts[perm]


def any_neighbor(mask: np.ndarray, periodic_x: bool) -> np.ndarray:
    """True where some 8-neighbour (self excluded) is true.  grid.py:59-76."""
    H, W = mask.shape
    padded = np.zeros((H + 2, W + 2), dtype=bool)
    padded[1:H + 1, 1:W + 1] = mask
    if periodic_x:
        padded[1:H + 1, 0] = mask[:, W - 1]
        padded[1:H + 1, W + 1] = mask[:, 0]
    hit = np.zeros((H, W), dtype=bool)
    for oy in range(3):
        for ox in range(3):
            if ox != 1 or oy != 1:
                hit |= padded[oy:oy + H, ox:ox + W]
    return hit


def active_mask(lab: np.ndarray, periodic_x: bool) -> np.ndarray:
    """Inpaint pixels with a Readable 8-neighbour.  grid.py:104-106."""
    return (lab == INPAINT) & any_neighbor(lab == READABLE, periodic_x)


def inner_mask(lab: np.ndarray, periodic_x: bool = False) -> np.ndarray:
    """grid.py:84-88 (mask form)."""
    inp = lab == INPAINT
    return inp & any_neighbor(~inp, periodic_x)


def outer_mask(lab: np.ndarray, periodic_x: bool = False) -> np.ndarray:
    """grid.py:91-95 (mask form)."""
    inp = lab == INPAINT
    return ~inp & any_neighbor(inp, periodic_x)


# ------------------------------------------------------------ ball sampler

def ball_points(g: np.ndarray, offs: np.ndarray, rotated: bool) -> np.ndarray:
    """Relative sample points (F, K, 2) from guide rows g (F, 2).  engine.py:150-164."""
    count = g.shape[0]
    if not rotated:
        return np.broadcast_to(offs, (count,) + offs.shape)
    length = np.hypot(g[:, 0], g[:, 1])
    is_zero = length == 0.0
    denom = np.where(is_zero, 1.0, length)
    ux = np.where(is_zero, 0.0, g[:, 0] / denom)
    uy = np.where(is_zero, 1.0, g[:, 1] / denom)
    n = offs[:, 0]
    m = offs[:, 1]
    px = n[None, :] * uy[:, None] + m[None, :] * ux[:, None]
    py = -n[None, :] * ux[:, None] + m[None, :] * uy[:, None]
    return np.stack([px, py], axis=-1)


def ball_weights(rel: np.ndarray, g: np.ndarray, mu: float, r: int) -> np.ndarray:
    """Eq. 3.2 weights; engine.py:131-147 (mu = inf: argmin-set rule)."""
    dist = np.hypot(rel[..., 0], rel[..., 1])
    gx = g[..., 0][..., None]
    gy = g[..., 1][..., None]
    if math.isinf(mu):
        length = np.sqrt(gx * gx + gy * gy)
        denom = np.where(length == 0.0, 1.0, length)
        d = (-gy * rel[..., 0] + gx * rel[..., 1]) / denom
        d2 = d * d
        tol = 1e-12 * max(1.0, float(r * r))
        chosen = d2 <= d2.min(axis=-1, keepdims=True) + tol
        return chosen / dist
    d = -gy * rel[..., 0] + gx * rel[..., 1]
    return np.exp(-(mu * mu) / (2.0 * float(r * r)) * d * d) / dist


def ghost_gather(img: np.ndarray, readable: np.ndarray, X: np.ndarray, Y: np.ndarray,
                 periodic_x: bool):
    """Strict bilinear ghost sampling, Eq. 3.3.  grid.py:158-211."""
    H, W = readable.shape
    C = img.shape[2]
    ix0 = np.floor(X).astype(np.int64)
    iy0 = np.floor(Y).astype(np.int64)
    tx = X - ix0
    ty = Y - iy0
    acc = np.zeros(X.shape + (C,))
    good = np.ones(X.shape, dtype=bool)
    img_rows = img.reshape(-1, C)
    read_flat = readable.reshape(-1)
    for cx, wx in ((ix0, 1.0 - tx), (ix0 + 1, tx)):
        for cy, wy in ((iy0, 1.0 - ty), (iy0 + 1, ty)):
            wc = wx * wy
            live = wc != 0.0
            if periodic_x:
                col = np.mod(cx, W)
                inside = (cy >= 0) & (cy < H)
            else:
                col = cx
                inside = (cx >= 0) & (cx < W) & (cy >= 0) & (cy < H)
            flat = np.where(inside, cy * W + col, 0)
            good &= (inside & read_flat[flat]) | ~live
            acc += np.where(live & inside, wc, 0.0)[..., None] * img_rows[flat]
    acc[~good] = 0.0
    return acc, good


def sample_frontier(u, readable, fx, fy, g, params, offs):
    """Weighted ball average, readable mass, total mass.  engine.py:175-199."""
    rotated = params.neighborhood == "rotated_ball"
    if g.ndim == 1:
        rel = ball_points(g[None, :], offs, rotated)[0]
        w = ball_weights(rel, g, params.mu, params.r)[None, :]
        X = fx[:, None] + rel[None, :, 0]
        Y = fy[:, None] + rel[None, :, 1]
    else:
        rel = ball_points(g, offs, rotated)
        w = ball_weights(rel, g, params.mu, params.r)
        X = fx[:, None] + rel[..., 0]
        Y = fy[:, None] + rel[..., 1]
    vals, ok = ghost_gather(u, readable, X, Y, params.periodic_x)
    wr = np.where(ok, w, 0.0)
    rmass = wr.sum(axis=1)
    tmass = (w * np.ones_like(ok, dtype=np.float64)).sum(axis=1)
    num = np.einsum("fk,fkc->fc", wr, vals)
    with np.errstate(invalid="ignore", divide="ignore"):
        avg = num / rmass[:, None]
    avg[rmass == 0.0] = 0.0
    return avg, rmass, tmass


def point_sample(u, labels, point, g, params):
    """Single-pixel (values, readable_mass, total_mass).  engine.py:202-221."""
    offs = disk_offsets(params.r)[1:]
    readable = labels == READABLE
    fx = np.array([float(point[0])])
    fy = np.array([float(point[1])])
    return sample_frontier(u, readable, fx, fy, np.asarray(g, dtype=np.float64), params, offs)


# --------------------------------------------------------------- fill loop

def _smooth(arr, s):
    """guide.py:46-48."""
    return ndimage.gaussian_filter(arr, sigma=s, truncate=2.0, mode="constant", cval=0.0)


def tensor_field(image, indicator, sigma, rho):
    """guide.py:91-120: indicator-weighted structure tensor (J11, J12, J22, mass_r)."""
    ind = indicator.astype(np.float64)
    mass_s = _smooth(ind, sigma)
    safe_s = np.where(mass_s > 0.0, mass_s, 1.0)
    J11 = np.zeros(ind.shape)
    J12 = np.zeros(ind.shape)
    J22 = np.zeros(ind.shape)
    for ch in range(image.shape[2]):
        v = _smooth(ind * image[:, :, ch], sigma) / safe_s
        gy, gx = np.gradient(v)
        J11 += gx * gx
        J12 += gx * gy
        J22 += gy * gy
    J11 *= ind
    J12 *= ind
    J22 *= ind
    mass_r = _smooth(ind, rho)
    safe_r = np.where(mass_r > 0.0, mass_r, 1.0)
    return (_smooth(J11, rho) / safe_r, _smooth(J12, rho) / safe_r,
            _smooth(J22, rho) / safe_r, mass_r)


def coherence_directions(image, readable, ix, iy, sigma=2.0, rho=4.0, lam=1e-5):
    """guide.py:330-355 (crop to the queries' box + cascade_radius + 2, guide.py:60-62),
    eigen split guide.py:123-136."""
    ix = np.asarray(ix)
    iy = np.asarray(iy)
    H, W = readable.shape
    pad = int(math.ceil(2.0 * sigma + 2.0 * rho)) + 2
    j0 = max(0, int(iy.min()) - pad)
    j1 = min(H, int(iy.max()) + pad + 1)
    i0 = max(0, int(ix.min()) - pad)
    i1 = min(W, int(ix.max()) + pad + 1)
    J11, J12, J22, mass_r = tensor_field(image[j0:j1, i0:i1], readable[j0:j1, i0:i1], sigma, rho)
    qj = iy - j0
    qi = ix - i0
    a, b, c = J11[qj, qi], J12[qj, qi], J22[qj, qi]
    mean = (a + c) / 2.0
    disc = np.sqrt(((a - c) / 2.0) ** 2 + b * b)
    phi = 0.5 * np.arctan2(2.0 * b, a - c)
    lo, hi, vx, vy = mean - disc, mean + disc, -np.sin(phi), np.cos(phi)
    coh = np.tanh((hi - lo) / lam)
    g = np.stack([coh * vx, coh * vy], axis=-1)
    g[mass_r[qj, qi] <= 0.0] = 0.0
    return g


def _frontier_g(params, guide_vecs, frontier, u=None, lab=None):
    """engine.py:234-249."""
    if params.g_source == "fixed":
        gf = params.g_fixed or (0.0, 0.0)
        return np.array([float(gf[0]), float(gf[1])])
    if params.g_source == "guide_field":
        if guide_vecs is None:
            return np.zeros(2)
        return guide_vecs.reshape(-1, 2)[frontier]
    iy, ix = np.divmod(frontier, lab.shape[1])
    return coherence_directions(u, lab == READABLE, ix, iy, sigma=params.sigma,
                                rho=params.rho, lam=params.coherence_lambda)


def _neighbor_mean(u, readable, idx, W, periodic_x):
    """engine.py:252-267."""
    H = readable.shape[0]
    j, i = divmod(idx, W)
    acc = np.zeros(u.shape[2])
    cnt = 0
    for di, dj in NEIGHBOR_OFFSETS:
        ii, jj = i + di, j + dj
        if periodic_x:
            ii %= W
        if 0 <= ii < W and 0 <= jj < H and readable[jj, ii]:
            acc += u[jj, ii]
            cnt += 1
    return None if cnt == 0 else acc / cnt


def _paint_unfillable(u, lab, readable):
    """Nearest-readable colour for stranded Inpaint pixels.  engine.py:270-283."""
    stranded = lab == INPAINT
    count = int(stranded.sum())
    if count == 0:
        return 0, stranded
    if readable.any():
        _, (jn, in_) = ndimage.distance_transform_edt(~readable, return_indices=True)
        jr, ir = np.nonzero(stranded)
        u[jr, ir] = u[jn[jr, ir], in_[jr, ir]]
    else:
        u[stranded] = 0.5
    lab[stranded] = READABLE
    return count, stranded


def _tracked_update(frontier, fill, filled_idx, lab, periodic_x):
    """Survivors + Inpaint 8-neighbours of the filled pixels, sorted.

    tracker.py:42-79 (``_active_filter`` is kept: it is part of the
    reference's per-shell work even though it never removes a candidate).
    """
    H, W = lab.shape
    flat = lab.reshape(-1)
    survivors = frontier[~fill]
    jy, ix = np.divmod(filled_idx, W)
    grown = []
    for di, dj in NEIGHBOR_OFFSETS:
        ii = ix + di
        jj = jy + dj
        if periodic_x:
            ii = np.mod(ii, W)
            ok = (jj >= 0) & (jj < H)
        else:
            ok = (ii >= 0) & (ii < W) & (jj >= 0) & (jj < H)
        nb = jj * W + np.where(ok, ii, 0)
        live = ok & (flat[np.where(ok, nb, 0)] == INPAINT)
        grown.append(nb[live])
    pool = np.concatenate([survivors] + grown)
    cand = np.unique(pool)
    # active filter, tracker.py:59-66
    cy, cx = np.divmod(cand, W)
    keep = flat[cand] == INPAINT
    has_read = np.zeros(cand.size, dtype=bool)
    for di, dj in NEIGHBOR_OFFSETS:
        ii = cx + di
        jj = cy + dj
        if periodic_x:
            ii = np.mod(ii, W)
            ok = (jj >= 0) & (jj < H)
        else:
            ok = (ii >= 0) & (ii < W) & (jj >= 0) & (jj < H)
        nb = jj * W + np.where(ok, ii, 0)
        has_read |= ok & (flat[np.where(ok, nb, 0)] == READABLE)
    return int(cand.size), cand[keep & has_read]


def fill(image, labels, guide=None, params=None, tracked: bool = True):
    """Run Algorithm 1.  engine.py:286-376 with the tracker hook tracker.py:161-170.

    Returns a dict with keys ``u`` (H, W, C) float64, ``rows`` (list of
    (iteration, frontier_size, candidates, threads, filled)), ``iterations``,
    ``filled``, ``deadlock_fills``, ``unfillable``, ``unfillable_count``,
    ``enter`` and ``fillshell`` (int32 (H, W)).
    """
    H, W = labels.shape
    u = np.ascontiguousarray(image, dtype=np.float64).copy()
    lab = labels.copy()
    guide_vecs = None if guide is None else np.asarray(guide, dtype=np.float64)
    readable = lab == READABLE
    hull = None
    if bool(readable.any()):
        seed = u[readable]
        hull = (float(seed.min()), float(seed.max()))
    remaining = int((lab == INPAINT).sum())
    offs = disk_offsets(params.r)[1:]
    data_term_live = params.order == "smart_with_data_term"
    frontier = np.flatnonzero(active_mask(lab, params.periodic_x))

    enter = np.full(H * W, -1, dtype=np.int32)
    fillshell = np.full(H * W, -1, dtype=np.int32)
    enter[frontier] = 0

    read_flat = readable.reshape(-1)
    lab_flat = lab.reshape(-1)
    u_rows = u.reshape(-1, u.shape[2])
    out = dict(rows=[], deadlock_fills=0, filled=0, unfillable=False, unfillable_count=0)

    k = 0
    while remaining > 0:
        if frontier.size == 0:
            out["unfillable"] = True
            cnt, stranded = _paint_unfillable(u, lab, readable)
            out["unfillable_count"] = cnt
            fillshell[stranded.reshape(-1)] = -2
            break
        g = _frontier_g(params, guide_vecs, frontier, u, lab)
        fy, fx = np.divmod(frontier, W)
        vals, rw, tw = sample_frontier(u, readable, fx.astype(np.float64),
                                       fy.astype(np.float64), g, params, offs)
        conf = rw / tw
        if params.order == "onion":
            ready = np.ones(frontier.size, dtype=bool)
        elif params.order == "smart" or not data_term_live:
            ready = conf > params.c
        else:
            gnorm = np.hypot(g[..., 0], g[..., 1])
            if g.ndim == 1:
                gnorm = np.full(frontier.size, gnorm)
            if not (gnorm > 0.0).any():
                data_term_live = False
                ready = conf > params.c
            else:
                ready = (gnorm > params.c2) & (conf > params.c)
        fill_mask = ready & (rw > 0.0)
        if not fill_mask.any():
            best = int(np.argmax(conf))
            if rw[best] > 0.0:
                fill_mask[best] = True
            else:
                fb = _neighbor_mean(u, readable, int(frontier[best]), W, params.periodic_x)
                if fb is None:
                    out["unfillable"] = True
                    cnt, stranded = _paint_unfillable(u, lab, readable)
                    out["unfillable_count"] = cnt
                    fillshell[stranded.reshape(-1)] = -2
                    break
                vals[best] = fb
                fill_mask[best] = True
            out["deadlock_fills"] += 1

        filled_idx = frontier[fill_mask]
        u_rows[filled_idx] = vals[fill_mask]
        read_flat[filled_idx] = True
        lab_flat[filled_idx] = READABLE
        fillshell[filled_idx] = k
        remaining -= filled_idx.size
        out["filled"] += int(filled_idx.size)

        if tracked:
            cand, nxt = _tracked_update(frontier, fill_mask, filled_idx, lab, params.periodic_x)
            threads = int(frontier.size)
        else:
            cand = W * H
            threads = W * H
            nxt = np.flatnonzero(active_mask(lab, params.periodic_x))
        new = nxt[enter[nxt] < 0]
        enter[new] = k + 1
        out["rows"].append((k, int(frontier.size), int(cand), int(threads), int(filled_idx.size)))
        frontier = nxt
        k += 1

    out["iterations"] = k
    if hull is not None:
        np.clip(u, hull[0], hull[1], out=u)
    out["u"] = u
    out["enter"] = enter.reshape(H, W)
    out["fillshell"] = fillshell.reshape(H, W)
    return out


# ------------------------------------------------------------- guide field

def flatten_cubic(ctrl: np.ndarray, tol: float) -> np.ndarray:
    """Adaptive de Casteljau flattening of one cubic.  splines.py:53-73."""
    a, b, c, d = ctrl
    chord = d - a
    L = math.hypot(chord[0], chord[1])
    if L < 1e-12:
        dev = max(np.hypot(*(b - a)), np.hypot(*(c - a)))
    else:
        nrm = np.array([-chord[1], chord[0]]) / L
        dev = max(abs(float((b - a) @ nrm)), abs(float((c - a) @ nrm)))
    if dev <= tol:
        return np.stack([a, d])
    ab = (a + b) / 2
    bc = (b + c) / 2
    cd = (c + d) / 2
    abc = (ab + bc) / 2
    bcd = (bc + cd) / 2
    mid = (abc + bcd) / 2
    left = flatten_cubic(np.stack([a, ab, abc, mid]), tol)
    right = flatten_cubic(np.stack([mid, bcd, cd, d]), tol)
    return np.concatenate([left, right[1:]], axis=0)


def polyline(points: np.ndarray, kind: str, tol: float = 0.25) -> np.ndarray:
    """splines.py:42-50."""
    points = np.asarray(points, dtype=np.float64)
    if kind == "polyline":
        return points
    parts = [points[0:1]]
    for k in range(0, len(points) - 1, 3):
        parts.append(flatten_cubic(points[k:k + 4], tol)[1:])
    return np.concatenate(parts, axis=0)


def _polyline_distance(px, py, poly):
    """guide.py:286-300."""
    best = np.full(px.shape, np.inf)
    for s in range(len(poly) - 1):
        ax, ay = poly[s]
        bx, by = poly[s + 1]
        abx, aby = bx - ax, by - ay
        L2 = abx * abx + aby * aby
        if L2 == 0.0:
            d = np.hypot(px - ax, py - ay)
        else:
            t = np.clip(((px - ax) * abx + (py - ay) * aby) / L2, 0.0, 1.0)
            d = np.hypot(px - (ax + t * abx), py - (ay + t * aby))
        np.minimum(best, d, out=best)
    return best


def guide_field(polys, dirs, labels: np.ndarray, eta: float = 3.0) -> np.ndarray:
    """Nearest-spline Gaussian falloff field.  guide.py:303-327.

    ``polys``: list of (P, 2) float64 polylines; ``dirs``: list of (dx, dy).
    """
    H, W = labels.shape
    out = np.zeros((H, W, 2))
    if len(polys) == 0:
        return out
    jj, ii = np.nonzero(labels == INPAINT)
    if jj.size == 0:
        return out
    px = ii.astype(np.float64)
    py = jj.astype(np.float64)
    dists = np.stack([_polyline_distance(px, py, np.asarray(p, dtype=np.float64)) for p in polys])
    near = np.argmin(dists, axis=0)
    dmin = dists[near, np.arange(px.size)]
    fall = np.exp(-(dmin * dmin) / (2.0 * eta * eta))
    fall[dmin > 3.0 * eta] = 0.0
    dv = np.array([[float(d[0]), float(d[1])] for d in dirs])
    out[jj, ii, 0] = dv[near, 0] * fall
    out[jj, ii, 1] = dv[near, 1] * fall
    return out


# ----------------------------------------------------------------- helpers

class Params:
    """Minimal stand-in for FillParams (engine.py:33-60) used by the oracle."""

    def __init__(self, r=3, mu=50.0, c=0.05, c2=0.0, order="smart",
                 neighborhood="rotated_ball", g_source="guide_field", g_fixed=None,
                 periodic_x=False, sigma=2.0, rho=4.0, coherence_lambda=1e-5):
        self.sigma = sigma
        self.rho = rho
        self.coherence_lambda = coherence_lambda
        self.r = r
        self.mu = mu
        self.c = c
        self.c2 = c2
        self.order = order
        self.neighborhood = neighborhood
        self.g_source = g_source
        self.g_fixed = g_fixed
        self.periodic_x = periodic_x

    @classmethod
    def of(cls, p):
        return cls(r=p.r, mu=p.mu, c=p.c, c2=p.c2, order=p.order,
                   neighborhood=p.neighborhood, g_source=p.g_source,
                   g_fixed=p.g_fixed, periodic_x=p.periodic_x,
                   sigma=getattr(p, "sigma", 2.0), rho=getattr(p, "rho", 4.0),
                   coherence_lambda=getattr(p, "coherence_lambda", 1e-5))


def numpy_exp_flavour() -> str:
    """Which float64 exp numpy dispatches to on this host.

    AVX512_SKX hosts run Intel SVML ``__svml_exp8_ha`` (the flavour the CUDA
    engine reproduces bit for bit); other hosts call libm ``exp``.
    """
    try:
        from numpy._core import _multiarray_umath as m
        feats = m.__cpu_features__
    except Exception:  # pragma: no cover
        return "unknown"
    return "svml" if feats.get("AVX512_SKX") else "libm"
