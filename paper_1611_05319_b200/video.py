"""Frame-parallel video fill (BASELINE.json config C5).

Frames of a video are independent fills, so a batch is
partitioned into contiguous frame blocks, one block per GPU / rank, with no
data-path collective: every rank fills its block with one batched
gf_fill_splines launch.  Collectives are used only for bookkeeping (the
max-over-ranks timing, optional result gathers), never inside the fill.
"""

from __future__ import annotations

import numpy as np


def frame_block(n_frames: int, world: int, rank: int) -> range:
    """Contiguous block of frames owned by ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def frame_checksum(u: np.ndarray) -> float:
    """Order-independent digest used to compare per-frame results across ranks."""
    return float(np.asarray(u, dtype=np.float64).sum())


def fill_video(images, labels, splines, params, tracked=True, device=None, workspace=None):
    """Fill a (N, H, W, C) batch of frames that share one spline set.

    images: float32/float64 CUDA tensor (N, H, W, C); labels: uint8 CUDA
    tensor (N, H, W); splines: a ``_device.SegmentSet`` or None (g = 0).
    Returns the ``fill_device`` result dict (out, stats, rows, ...).
    """
    from ._device import fill_device

    return fill_device(images, labels, None, params, tracked=tracked, splines=splines,
                       workspace=workspace)
