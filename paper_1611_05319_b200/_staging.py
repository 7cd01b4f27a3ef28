"""Host <-> device transfers for the numpy drop-in API.

The reference API takes and returns host float64 arrays (1080p RGB = 50 MB
each way).  Pageable copies are slow (measured on the B200 box: H2D 3.5 ms,
D2H 23.5 ms for 50 MB), pinned ones ~0.9 ms.  The stager keeps cached
pinned staging buffers and moves data in chunks: host threads copy chunk i
into / out of pinned memory while the DMA engine moves chunk i-1 (numpy's
copyto releases the GIL, so the host copies run in parallel).
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_CHUNK = 8 << 20
# below this a plain pageable .to() is faster than the threaded stager
# (B200 box, 2 MB labels: 0.13 ms direct vs 0.37 ms staged)
_STAGE_MIN = 4 << 20
_lock = threading.Lock()
_pool = None
_pinned = {}


def _executor():
    global _pool
    with _lock:
        if _pool is None:
            _pool = ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1)))
        return _pool


def _staging(nbytes: int, slot: str):
    """Cached pinned uint8 buffer of at least nbytes, one per (slot, calling
    thread): concurrent fills from several host threads never share one."""
    import torch

    key = (slot, threading.get_ident())
    with _lock:
        buf = _pinned.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
            _pinned[key] = buf
        return buf


def _chunks(n: int):
    return [(o, min(n, o + _CHUNK)) for o in range(0, n, _CHUNK)]


def upload(arr: np.ndarray, device, slot: str = "up"):
    """numpy array -> CUDA tensor of the same dtype/shape (stream-ordered)."""
    import torch

    a = np.ascontiguousarray(arr)
    n = a.nbytes
    dst = torch.empty(a.shape, dtype=torch.from_numpy(a[:0].reshape(-1)).dtype, device=device)
    if n == 0:
        return dst
    if n < _STAGE_MIN:
        return torch.from_numpy(a).to(device)
    ta = torch.from_numpy(a.reshape(-1).view(np.uint8))
    if ta.is_pinned():
        # already in page-locked memory (e.g. an array this package returned):
        # one DMA, no staging copy
        # (stream-ordered; every public entry synchronises before it returns)
        dst.view(-1).view(torch.uint8).copy_(ta, non_blocking=True)
        return dst
    stage = _staging(n, slot)
    src = a.reshape(-1).view(np.uint8)
    host = stage.numpy()
    dflat = dst.view(-1).view(torch.uint8)
    stream = torch.cuda.current_stream()
    futs = [_executor().submit(np.copyto, host[lo:hi], src[lo:hi]) for lo, hi in _chunks(n)]
    for (lo, hi), fut in zip(_chunks(n), futs):
        fut.result()
        dflat[lo:hi].copy_(stage[lo:hi], non_blocking=True)
    # the staging buffer is reused by the next call: wait for the DMA
    stream.synchronize()
    return dst


class _BufferOwner:
    """Owner of one pooled pinned buffer, exposed to numpy through
    ``__array_interface__``.  Every array made from it -- and every view of
    such an array, whose ``.base`` numpy collapses to this object -- keeps it
    alive, so the buffer goes back to the pool only when the last user is
    gone (not when the first returned array dies)."""

    __slots__ = ("buf", "__array_interface__", "__weakref__")

    def __init__(self, buf, n, shape, dtype):
        self.buf = buf
        self.__array_interface__ = {"shape": tuple(shape), "typestr": np.dtype(dtype).str,
                                    "data": (buf.data_ptr(), False), "version": 3}


class _PinnedPool:
    """Recycled pinned host buffers for returned arrays.

    ``take`` hands out a numpy array backed by pinned, already-touched memory,
    so steady-state calls pay neither page faults nor pinned allocation, and
    the D2H lands in it at full DMA speed.  The buffer returns to the pool
    when its ``_BufferOwner`` dies: every numpy view references the owner,
    and tensors from ``take_tensor`` hold the numpy array (torch.from_numpy),
    so a live view of a result can never see its memory reused.
    """

    def __init__(self):
        self.free = {}
        self.lock = threading.Lock()

    @staticmethod
    def _alloc(n):
        import torch

        return torch.empty(max(n, 1), dtype=torch.uint8, pin_memory=True)

    def take(self, shape, dtype):
        import weakref

        dtype = np.dtype(dtype)
        n = int(np.prod(shape)) * dtype.itemsize
        with self.lock:
            lst = self.free.get(n)
            buf = lst.pop() if lst else None
        if buf is None:
            buf = self._alloc(n)
        owner = _BufferOwner(buf, n, shape, dtype)
        arr = np.asarray(owner)
        weakref.finalize(owner, self._give, n, buf)
        return arr, buf

    def take_tensor(self, shape, dtype):
        """Like ``take``, as a pinned CPU torch tensor.  The tensor's storage
        holds the numpy array (hence the owner): the buffer is recycled only
        after every tensor view is released."""
        import torch

        np_dtype = torch.empty(0, dtype=dtype).numpy().dtype
        arr, buf = self.take(shape, np_dtype)
        return torch.from_numpy(arr), buf

    def _give(self, n, buf):
        with self.lock:
            lst = self.free.setdefault(n, [])
            if len(lst) < 4:
                lst.append(buf)


_pool_out = _PinnedPool()


def download(t) -> np.ndarray:
    """CUDA tensor -> new numpy array (synchronous), DMA'd straight into a
    recycled pinned buffer."""
    import torch

    t = t.contiguous()
    dtype = torch.empty(0, dtype=t.dtype).numpy().dtype
    if t.numel() * dtype.itemsize < (1 << 20):
        return t.cpu().numpy()
    out, buf = _pool_out.take(tuple(t.shape), dtype)
    buf[: out.nbytes].copy_(t.view(-1).view(torch.uint8), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out


def download_tensor(t):
    """CUDA tensor -> new pinned CPU tensor (synchronous, recycled buffer)."""
    import torch

    t = t.contiguous()
    out, buf = _pool_out.take_tensor(tuple(t.shape), t.dtype)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out


_report_buf = {}


def read_report(stats, rows, max_rows=4096):
    """One pinned read-back of a frame's stats and its first report rows
    (a single synchronisation instead of two)."""
    import torch

    n_rows = min(rows.shape[0], max_rows)
    key = (stats.numel(), n_rows, threading.get_ident())
    with _lock:
        buf = _report_buf.get(key)
        if buf is None:
            buf = (torch.empty(stats.numel(), dtype=torch.int32, pin_memory=True),
                   torch.empty((n_rows, 2), dtype=torch.int32, pin_memory=True))
            _report_buf[key] = buf
    buf[0].copy_(stats.reshape(-1), non_blocking=True)
    buf[1].copy_(rows[:n_rows], non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return buf[0].numpy().copy(), buf[1].numpy().copy()


# ------------------------------------------------------------- mirrored path
#
# A fill leaves every Readable pixel bit-identical (engine.py:364-376), so the
# result buffer is seeded with the INPUT by device->host DMA chunk by chunk as
# the upload lands (the two directions of the link run concurrently), and after
# the fill gf_output_delta writes only the changed pixels into it over the
# mapped pinned mapping.  The full-frame download leaves the critical path.

_MIRROR_CHUNK = 8 << 20  # DMA piece size (B200 box: 2 MB 1.76 ms, 8 MB 1.48 ms per C2 frame)
_side = {}
_mirror_ok = {}


def _side_stream(device):
    import torch

    key = (str(device), threading.get_ident())
    with _lock:
        s = _side.get(key)
        if s is None:
            s = torch.cuda.Stream(device=device)
            _side[key] = s
        return s


def mirror_supported(device) -> bool:
    """Whether pinned host buffers are device-writable here (UVA mapping);
    probed once per device with a one-pixel gf_output_delta."""
    import ctypes

    import torch

    from . import _native as N

    key = str(device)
    ok = _mirror_ok.get(key)
    if ok is None:
        lib = N.load()
        a = torch.zeros(1, dtype=torch.float32, device=device)
        b = torch.ones(1, dtype=torch.float32, device=device)
        h = torch.zeros(1, dtype=torch.float32, pin_memory=True)
        rc = lib.gf_output_delta(1, 1, N.GF_F32, ctypes.c_void_p(a.data_ptr()),
                                 ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(h.data_ptr()),
                                 None, N.stream_ptr())
        torch.cuda.current_stream().synchronize()
        ok = rc == N.GF_OK and float(h[0]) == 1.0
        _mirror_ok[key] = ok
    return ok


class Mirror:
    """Device copy of a host frame plus its host result buffer, seeded with
    the input by the side stream as the upload proceeds."""

    def __init__(self, device, shape, dtype_t, as_tensor: bool):
        import torch

        self.device = device
        self.side = _side_stream(device)
        itemsize = torch.empty(0, dtype=dtype_t).element_size()
        if as_tensor:
            self.result, self.buf = _pool_out.take_tensor(shape, dtype_t)
        else:
            np_dtype = torch.empty(0, dtype=dtype_t).numpy().dtype
            self.result, self.buf = _pool_out.take(shape, np_dtype)
        self.nbytes = int(np.prod(shape)) * itemsize

    def upload(self, host_ptr, dev_ptr, lo, hi):
        """H2D of bytes [lo, hi) on the current stream; each landed piece is
        mirrored D2H into the result buffer on the side stream (C loop:
        gf_upload_mirrored, a few us of host work per piece)."""
        import ctypes

        from . import _native as N

        N.check(N.load().gf_upload_mirrored(
            ctypes.c_void_p(host_ptr + lo), ctypes.c_void_p(dev_ptr + lo),
            ctypes.c_void_p(self.buf.data_ptr() + lo), hi - lo, _MIRROR_CHUNK, N.stream_ptr(),
            ctypes.c_void_p(self.side.cuda_stream)))

    def settle(self):
        """Error path: let every transfer touching the result buffer land
        (the side stream's mirror, and the current stream's H2D reads and
        delta writes) before the buffer can go back to the pool."""
        import torch

        for s in (self.side, torch.cuda.current_stream()):
            try:
                s.synchronize()
            except Exception:
                pass

    def finish(self, d_in, d_out):
        """Enqueue the delta write on the current stream (after the mirror);
        the caller's next synchronisation makes ``result`` final."""
        import ctypes

        import torch

        from . import _native as N

        main = torch.cuda.current_stream()
        main.wait_stream(self.side)
        d_in.record_stream(self.side)
        C = d_in.shape[-1]
        n_px = d_in.numel() // C
        dt = N.GF_F64 if d_in.dtype == torch.float64 else N.GF_F32
        N.check(N.load().gf_output_delta(n_px, C, dt, ctypes.c_void_p(d_in.data_ptr()),
                                         ctypes.c_void_p(d_out.data_ptr()),
                                         ctypes.c_void_p(self.buf.data_ptr()), None,
                                         N.stream_ptr()))


def upload_mirrored(src, device, as_tensor: bool):
    """Host frame (numpy array, or pinned CPU tensor) -> (CUDA tensor, Mirror).

    Pinned sources are DMA'd straight from the caller's memory and each
    landed chunk is mirrored back into the result buffer on the side stream.
    Pageable numpy arrays are copied by host threads into the result buffer
    itself, which then serves as the H2D source (no mirror needed).
    """
    import torch

    if as_tensor:
        t = src
        dst = torch.empty(t.shape, dtype=t.dtype, device=device)
        mir = Mirror(device, tuple(t.shape), t.dtype, True)
        mir.upload(t.data_ptr(), dst.data_ptr(), 0, mir.nbytes)
        return dst, mir
    a = np.ascontiguousarray(src)
    n = a.nbytes
    dst = torch.empty(a.shape, dtype=torch.from_numpy(a[:0].reshape(-1)).dtype, device=device)
    mir = Mirror(device, a.shape, dst.dtype, False)
    if torch.from_numpy(a.reshape(-1).view(np.uint8)).is_pinned():
        # page-locked numpy memory (e.g. a result of this package): DMA directly
        mir.upload(a.ctypes.data, dst.data_ptr(), 0, n)
        return dst, mir
    # pageable memory: the host threads copy the frame straight into the
    # pinned RESULT buffer, chunk by chunk, and each landed chunk is DMA'd to
    # the device from there.  The result is then already seeded with the
    # input (no D2H mirror), and host memory carries 150 MB per 1080p f64
    # frame instead of 200 (copy into a staging buffer, H2D from it, D2H
    # into the result) -- the bound of this path on the B200 box.
    srcb = a.reshape(-1).view(np.uint8)
    host = mir.buf.numpy()
    dflat = dst.view(-1).view(torch.uint8)
    # (smaller copy pieces than the DMA chunk measured slower: future and
    # GIL overhead; tools/exp_numpy_ab.sh)
    parts = _chunks_of(n, _CHUNK)
    futs = [_executor().submit(np.copyto, host[lo:hi], srcb[lo:hi]) for lo, hi in parts]
    for (lo, hi), fut in zip(parts, futs):
        fut.result()
        dflat[lo:hi].copy_(mir.buf[lo:hi], non_blocking=True)
    return dst, mir


def _chunks_of(n: int, size: int):
    return [(o, min(n, o + size)) for o in range(0, n, size)]
