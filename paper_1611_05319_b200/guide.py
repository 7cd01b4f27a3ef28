"""Guide field from splines -- drop-in for the reference's build_guide_field.

``build_guide_field`` (guide.py:303-327) runs the GPU rasteriser
(gf_guide_field): per Inpaint pixel, the minimum distance to each spline's
flattened polyline, the first nearest spline, and the Gaussian falloff
g = dir * exp(-d^2 / (2 eta^2)), zero beyond 3 eta and outside D.

``coherence_directions`` (guide.py:330-355) runs the masked structure tensor
on the device (gf_coherence_directions).  Automatic spline detection
(guide.py:55-283: measurement ring, Canny edge seeds, ray tracing) is outside
the accelerated path and raises NotImplementedError.
"""

from __future__ import annotations

import numpy as np

from .grid import INPAINT

DEFAULT_SIGMA = 2.0
DEFAULT_RHO = 4.0
DEFAULT_LAMBDA = 1e-5
DEFAULT_ETA = 3.0


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


def detect_splines(image, labels, *args, **kwargs):
    """Auto spline detection is not on the B200 path (needs Canny)."""
    raise NotImplementedError(
        "automatic spline detection (guide.py:270-283) is outside the accelerated fill path; "
        "pass user splines to build_guide_field")


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
