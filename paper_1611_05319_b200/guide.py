"""Guide field from splines -- drop-in for the reference's build_guide_field.

``build_guide_field`` (guide.py:303-327) runs the GPU rasteriser
(gf_guide_field): per Inpaint pixel, the minimum distance to each spline's
flattened polyline, the first nearest spline, and the Gaussian falloff
g = dir * exp(-d^2 / (2 eta^2)), zero beyond 3 eta and outside D.

Automatic spline detection (guide.py:55-283: measurement ring, Canny edge
seeds, structure tensor, ray tracing) and the coherence-transport g source
(guide.py:330-355) are outside the accelerated path (SURVEY.md section
8f-1/8f-2) and raise NotImplementedError here.
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


def coherence_directions(*args, **kwargs):
    raise NotImplementedError("coherence-transport directions are outside the accelerated path")
