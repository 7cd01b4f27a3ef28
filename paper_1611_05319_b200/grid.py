"""Label lattice conventions and lattice operators (reference grid.py).

Conventions are the reference's (grid.py:1-16): images (H, W, C) in [0, 1],
labels uint8 in {READABLE=0, BYSTANDER=128, INPAINT=255}, pixel (i, j) =
(column, row), arrays indexed [j, i], flat index j*W + i.

The lattice scans (boundary masks, ghost sampling) run on the GPU through
the C ABI; the tiny geometric helpers (disk offsets, rotation matrices)
stay on the host because they are O(r^2) constants.
"""

from __future__ import annotations

import numpy as np

READABLE = 0
BYSTANDER = 128
INPAINT = 255

_LABEL_VALUES = (READABLE, BYSTANDER, INPAINT)

# (di, dj), the reference's fixed order (grid.py:29-33)
NEIGHBOR_OFFSETS = (
    (-1, -1), (0, -1), (1, -1),
    (-1, 0), (1, 0),
    (-1, 1), (0, 1), (1, 1),
)


_LUT = np.ones(256, dtype=bool)
_LUT[list(_LABEL_VALUES)] = False


def validate_labels(labels, device_labels=None) -> None:
    """ValueError unless labels is 2-D over the three label values (grid.py:36-46).

    With ``device_labels`` (the same mask already on the GPU) the scan runs
    on the device; the host only locates the first bad value for the message.
    """
    labels = np.asarray(labels)
    if labels.ndim != 2:
        raise ValueError(f"label mask must be 2-D, got shape {labels.shape}")
    if device_labels is not None and labels.dtype == np.uint8:
        d = device_labels
        if not bool(((d != READABLE) & (d != BYSTANDER) & (d != INPAINT)).any()):
            return
    if labels.dtype == np.uint8:
        bad = _LUT[labels]
    else:
        bad = ~np.isin(labels, _LABEL_VALUES)
    if bad.any():
        j, i = np.nonzero(bad)
        raise ValueError(
            f"label mask holds value {int(labels[j[0], i[0]])} at (i={int(i[0])}, j={int(j[0])}); "
            f"allowed values are {_LABEL_VALUES}"
        )


def validate_image(image) -> None:
    """ValueError unless image is (H, W, C<=4) float, finite, in [0, 1] (grid.py:49-56)."""
    image = np.asarray(image)
    if image.ndim != 3 or image.shape[2] not in (1, 2, 3, 4):
        raise ValueError(f"image must be (H, W, C) with 1..4 channels, got shape {image.shape}")
    if not np.isfinite(image).all():
        raise ValueError("image holds non-finite values")
    if image.min() < 0.0 or image.max() > 1.0:
        raise ValueError("image values must lie in [0, 1]")


def _to_dev_labels(labels):
    import torch
    from . import _native as N

    dev = N.require_cuda()
    return torch.from_numpy(np.ascontiguousarray(labels, dtype=np.uint8)).to(dev)


def _masks(labels, periodic_x):
    from ._device import boundary_device

    validate_labels(labels)
    act, inn, out = boundary_device(_to_dev_labels(labels), periodic_x)
    return act.bool().cpu().numpy(), inn.bool().cpu().numpy(), out.bool().cpu().numpy()


def _coords(mask) -> set:
    j, i = np.nonzero(mask)
    return set(zip(i.tolist(), j.tolist()))


def active_boundary_mask(labels, periodic_x: bool = False) -> np.ndarray:
    """Inpaint pixels with a Readable 8-neighbour (grid.py:104-106), on the GPU."""
    return _masks(labels, periodic_x)[0]


def inner_boundary(labels, periodic_x: bool = False) -> set:
    """Inpaint pixels with a non-Inpaint 8-neighbour (grid.py:84-88)."""
    return _coords(_masks(labels, periodic_x)[1])


def outer_boundary(labels, periodic_x: bool = False) -> set:
    """Non-Inpaint pixels with an Inpaint 8-neighbour (grid.py:91-95)."""
    return _coords(_masks(labels, periodic_x)[2])


def active_boundary(labels, periodic_x: bool = False) -> set:
    """Set form of active_boundary_mask (grid.py:98-101)."""
    return _coords(_masks(labels, periodic_x)[0])


def offsets_in_disk(r: int) -> np.ndarray:
    """(n, m) with n^2 + m^2 <= r^2 in the reference's scan order, centre first (grid.py:109-124)."""
    if r < 1:
        raise ValueError("ball radius must be >= 1")
    pts = [(0.0, 0.0)]
    for m in range(-r, r + 1):
        for n in range(-r, r + 1):
            if n * n + m * m <= r * r and (n, m) != (0, 0):
                pts.append((float(n), float(m)))
    return np.asarray(pts, dtype=np.float64)


def rotation_to(g) -> np.ndarray:
    """Rotation mapping (0, 1) onto the direction of g; identity for g = 0 (grid.py:127-135)."""
    gx, gy = float(g[0]), float(g[1])
    norm = np.hypot(gx, gy)
    if norm == 0.0:
        return np.eye(2)
    ux, uy = gx / norm, gy / norm
    return np.array([[uy, ux], [-ux, uy]])


def rotated_ball(center, g, r: int) -> np.ndarray:
    """Ball points center + R(n, m) (grid.py:138-150)."""
    pts = offsets_in_disk(r) @ rotation_to(g).T
    pts[:, 0] += float(center[0])
    pts[:, 1] += float(center[1])
    return pts


def axis_ball(center, r: int) -> np.ndarray:
    """Axis-aligned lattice ball (grid.py:153-155)."""
    return rotated_ball(center, (0.0, 0.0), r)


def bilinear_gather(image, readable, X, Y, periodic_x: bool = False):
    """Strict ghost-point sampling on the GPU (grid.py:158-211).

    ``readable`` is a boolean (H, W) mask.  Returns (values X.shape + (C,),
    ok X.shape).
    """
    import torch
    from . import _native as N
    from ._device import bilinear_device

    dev = N.require_cuda()
    img = np.ascontiguousarray(image, dtype=np.float64)
    lab = np.where(np.asarray(readable, dtype=bool), READABLE, BYSTANDER).astype(np.uint8)
    Xb, Yb = np.broadcast_arrays(np.asarray(X, dtype=np.float64), np.asarray(Y, dtype=np.float64))
    shape = Xb.shape
    vals, ok = bilinear_device(torch.from_numpy(img).to(dev), torch.from_numpy(lab).to(dev),
                               torch.from_numpy(np.ascontiguousarray(Xb).reshape(-1)).to(dev),
                               torch.from_numpy(np.ascontiguousarray(Yb).reshape(-1)).to(dev),
                               periodic_x)
    C = img.shape[2]
    return vals.cpu().numpy().reshape(shape + (C,)), ok.bool().cpu().numpy().reshape(shape)


def sample_bilinear(image, readable, point, periodic_x: bool = False):
    """One ghost point: (values, True) or (None, False) (grid.py:214-221)."""
    vals, ok = bilinear_gather(image, readable, np.array([float(point[0])]),
                               np.array([float(point[1])]), periodic_x)
    if not ok[0]:
        return None, False
    return vals[0], True
