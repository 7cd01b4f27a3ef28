"""Image and label-mask files for the command line (reference fileio.py).

Formats (fileio.py:1-7 of the reference):
- images are 8-bit PNG, RGB or RGBA. Loading divides by 255 into float64.
  Saving clips to [0, 1] and rounds half away from zero (fileio.py:19-21),
  so values on a 0.5/255 boundary land the same way in both packages.
- label masks are binary (P5) or ASCII (P2) PGM with maxval 255 and the
  fixed encoding 0 / 128 / 255. They are read and written bit-exactly and
  validated with grid.validate_labels.

Host-side I/O only: the fill itself runs on the GPU.
"""

from __future__ import annotations

import numpy as np

from . import grid

_MODES = {1: "L", 2: "LA", 3: "RGB", 4: "RGBA"}


def to_uint8(values) -> np.ndarray:
    """[0, 1] floats -> uint8, round half away from zero (values are >= 0)."""
    return np.floor(np.clip(np.asarray(values, dtype=np.float64), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)


def load_image(path) -> np.ndarray:
    """PNG -> (H, W, C) float64 in [0, 1]; RGBA stays RGBA, everything else becomes RGB."""
    from PIL import Image

    with Image.open(path) as im:
        im = im if im.mode == "RGBA" else im.convert("RGB")
        arr = np.asarray(im, dtype=np.float64) / 255.0
    return arr[:, :, None] if arr.ndim == 2 else arr


def save_image(path, image) -> None:
    from PIL import Image

    image = np.asarray(image)
    grid.validate_image(image)
    data = to_uint8(image)
    mode = _MODES[data.shape[2]]
    Image.fromarray(data[:, :, 0] if data.shape[2] == 1 else data, mode=mode).save(path, format="PNG")


def _next_token(buf: bytes, pos: int):
    """Whitespace-delimited header token at or after ``pos`` ('#' comments skipped)."""
    n = len(buf)
    while pos < n:
        if buf[pos:pos + 1].isspace():
            pos += 1
        elif buf[pos:pos + 1] == b"#":
            nl = buf.find(b"\n", pos)
            pos = n if nl < 0 else nl + 1
        else:
            break
    end = pos
    while end < n and not buf[end:end + 1].isspace():
        end += 1
    if end == pos:
        raise ValueError("truncated PGM header")
    return buf[pos:end], end


def parse_labels(data: bytes) -> np.ndarray:
    """PGM bytes -> (H, W) uint8 labels (validated)."""
    magic, pos = _next_token(data, 0)
    if magic not in (b"P2", b"P5"):
        raise ValueError(f"not a PGM file: magic {magic!r}")
    fields = []
    for _ in range(3):
        tok, pos = _next_token(data, pos)
        fields.append(int(tok))
    width, height, maxval = fields
    if maxval != 255:
        raise ValueError(f"PGM maxval must be 255, got {maxval}")
    count = width * height
    if magic == b"P5":
        raster = data[pos + 1:pos + 1 + count]  # one whitespace byte ends the header
        if len(raster) < count:
            raise ValueError("PGM raster truncated")
        labels = np.frombuffer(raster, dtype=np.uint8).reshape(height, width).copy()
    else:
        values = data[pos:].split()[:count]
        if len(values) < count:
            raise ValueError("PGM raster truncated")
        labels = np.array([int(v) for v in values], dtype=np.int64)
        if labels.min() < 0 or labels.max() > 255:
            raise ValueError("PGM sample outside 0..255")
        labels = labels.astype(np.uint8).reshape(height, width)
    grid.validate_labels(labels)
    return labels


def load_labels(path) -> np.ndarray:
    with open(path, "rb") as fh:
        return parse_labels(fh.read())


def save_labels(path, labels) -> None:
    labels = np.asarray(labels)
    grid.validate_labels(labels)
    H, W = labels.shape
    with open(path, "wb") as fh:
        fh.write(f"P5\n{W} {H}\n255\n".encode("ascii"))
        fh.write(np.ascontiguousarray(labels, dtype=np.uint8).tobytes())
