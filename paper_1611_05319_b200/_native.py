"""ctypes binding of libgf_b200.so (the C ABI in include/guidefill_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1611_05319_b200/csrc``).  There is no fallback: if the
library or a CUDA device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GF_B200_LIB", os.path.join(_HERE, "libgf_b200.so"))

GF_OK = 0
GF_E_INVALID, GF_E_CUDA, GF_E_WORKSPACE, GF_E_UNSUPPORTED = -1, -2, -3, -4
GF_F32, GF_F64 = 0, 1
GF_ORDER = {"onion": 0, "smart": 1, "smart_with_data_term": 2}
GF_BALL = {"rotated_ball": 0, "axis_ball": 1}
GF_G_ZERO, GF_G_FIXED, GF_G_FIELD = 0, 1, 2
GF_MAX_RADIUS = 12
GF_STATS = 9
STAT_ITERATIONS, STAT_FILLED, STAT_DEADLOCK, STAT_UNFILLABLE = 0, 1, 2, 3
STAT_REMAINING, STAT_INPAINT, STAT_ROWS_OVERFLOW, STAT_LAST_FRONTIER = 4, 5, 6, 7
STAT_BAD_LABELS = 8

EXPORTS = (
    "gf_fill_workspace_bytes", "gf_fill_splines_workspace_bytes", "gf_fill", "gf_fill_splines",
    "gf_guide_field", "gf_sample_points",
    "gf_bilinear_gather", "gf_boundary_masks", "gf_output_delta", "gf_upload_mirrored",
    "gf_paint_unfillable_workspace_bytes", "gf_paint_unfillable",
    "gf_coherence_workspace_bytes", "gf_coherence_directions", "gf_frontier_candidates",
    "gf_commit_shell", "gf_structure_eigen", "gf_detect_workspace_bytes", "gf_detect_edges",
    "gf_trace_rays", "gf_last_error",
    "gf_abi_version", "gf_launch_count", "gf_host_exp", "gf_host_hypot", "gf_host_pairwise_sum",
    "gf_host_atan2", "gf_host_tanh", "gf_host_sincos", "gf_npmath_eval",
    "gf_coherence_fill_workspace_bytes", "gf_coherence_fill",
)


class FillParamsC(ctypes.Structure):
    _fields_ = [
        ("r", ctypes.c_int32),
        ("mu", ctypes.c_double),
        ("c", ctypes.c_double),
        ("c2", ctypes.c_double),
        ("order", ctypes.c_int32),
        ("neighborhood", ctypes.c_int32),
        ("g_mode", ctypes.c_int32),
        ("g_fixed", ctypes.c_double * 2),
        ("periodic_x", ctypes.c_int32),
        ("tracked", ctypes.c_int32),
    ]


class FramesC(ctypes.Structure):
    _fields_ = [
        ("n_frames", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("width", ctypes.c_int32),
        ("channels", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("image", ctypes.c_void_p),
        ("labels", ctypes.c_void_p),
        ("guide", ctypes.c_void_p),
        ("out", ctypes.c_void_p),
    ]


class FillOutputsC(ctypes.Structure):
    _fields_ = [
        ("frame_stats", ctypes.c_void_p),
        ("rows", ctypes.c_void_p),
        ("rows_cap", ctypes.c_int32),
        ("enter", ctypes.c_void_p),
        ("fillshell", ctypes.c_void_p),
        ("shell_trace", ctypes.c_void_p),
        ("trace_cap", ctypes.c_int32),
    ]


class SplinesC(ctypes.Structure):
    _fields_ = [
        ("n_seg", ctypes.c_int32),
        ("seg", ctypes.c_void_p),
        ("seg_spline", ctypes.c_void_p),
        ("n_splines", ctypes.c_int32),
        ("dirs", ctypes.c_void_p),
        ("eta", ctypes.c_double),
        ("frame_seg", ctypes.c_void_p),
    ]


class NativeError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


_lib = None


def load(required: bool = True):
    """Load the shared library once; raise if it is absent and required."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if required:
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        return None
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    lib.gf_fill_workspace_bytes.restype = ctypes.c_size_t
    lib.gf_fill_workspace_bytes.argtypes = [ctypes.POINTER(FramesC), ctypes.POINTER(FillParamsC)]
    lib.gf_fill.restype = ctypes.c_int
    lib.gf_fill.argtypes = [ctypes.POINTER(FramesC), ctypes.POINTER(FillParamsC),
                            ctypes.POINTER(FillOutputsC), P, ctypes.c_size_t, P]
    lib.gf_fill_splines_workspace_bytes.restype = ctypes.c_size_t
    lib.gf_fill_splines_workspace_bytes.argtypes = [ctypes.POINTER(FramesC),
                                                    ctypes.POINTER(FillParamsC),
                                                    ctypes.POINTER(SplinesC)]
    lib.gf_fill_splines.restype = ctypes.c_int
    lib.gf_fill_splines.argtypes = [ctypes.POINTER(FramesC), ctypes.POINTER(FillParamsC),
                                    ctypes.POINTER(SplinesC), ctypes.POINTER(FillOutputsC), P,
                                    ctypes.c_size_t, P]
    lib.gf_guide_field.restype = ctypes.c_int
    lib.gf_guide_field.argtypes = [ctypes.c_int32, ctypes.c_int32, P, ctypes.c_int32, P, P,
                                   ctypes.c_int32, P, ctypes.c_double, P, P]
    lib.gf_sample_points.restype = ctypes.c_int
    lib.gf_sample_points.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P,
                                     ctypes.c_int32, P, P, ctypes.POINTER(FillParamsC), P, P, P, P]
    lib.gf_bilinear_gather.restype = ctypes.c_int
    lib.gf_bilinear_gather.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P,
                                       ctypes.c_int32, P, P, ctypes.c_int32, P, P, P]
    lib.gf_boundary_masks.restype = ctypes.c_int
    lib.gf_boundary_masks.argtypes = [ctypes.c_int32, ctypes.c_int32, P, ctypes.c_int32, P, P, P, P]
    lib.gf_output_delta.restype = ctypes.c_int
    lib.gf_output_delta.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, P, P, P, P, P]
    lib.gf_upload_mirrored.restype = ctypes.c_int
    lib.gf_upload_mirrored.argtypes = [P, P, P, ctypes.c_int64, ctypes.c_int64, P, P]
    lib.gf_paint_unfillable_workspace_bytes.restype = ctypes.c_size_t
    lib.gf_paint_unfillable_workspace_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32]
    lib.gf_coherence_workspace_bytes.restype = ctypes.c_size_t
    lib.gf_coherence_workspace_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
    lib.gf_coherence_directions.restype = ctypes.c_int
    lib.gf_coherence_directions.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P,
                                            ctypes.c_int32, P, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_double, P, P, P, ctypes.c_size_t, P]
    lib.gf_frontier_candidates.restype = ctypes.c_int
    lib.gf_frontier_candidates.argtypes = [ctypes.c_int32, ctypes.c_int32, P, ctypes.c_int32,
                                           ctypes.c_int32, P, P, P, P]
    lib.gf_commit_shell.restype = ctypes.c_int
    lib.gf_commit_shell.argtypes = [ctypes.c_int32, ctypes.c_int32, P, P, P, P, P, ctypes.c_int32,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_int32, P, P, P, P,
                                    P, P]
    lib.gf_paint_unfillable.restype = ctypes.c_int
    lib.gf_paint_unfillable.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_int32, P, P, P, P, ctypes.c_size_t, P, P]
    lib.gf_structure_eigen.restype = ctypes.c_int
    lib.gf_structure_eigen.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P,
                                       ctypes.c_int32, P, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, P, P, ctypes.c_size_t, P]
    lib.gf_detect_workspace_bytes.restype = ctypes.c_size_t
    lib.gf_detect_workspace_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32]
    lib.gf_detect_edges.restype = ctypes.c_int
    lib.gf_detect_edges.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_int32, P, P, P, P, P, P,
                                    ctypes.c_size_t, P]
    lib.gf_trace_rays.restype = ctypes.c_int
    lib.gf_trace_rays.argtypes = [ctypes.c_int32, ctypes.c_int32, P, ctypes.c_int32, P, P,
                                  ctypes.c_double, P, P]
    lib.gf_last_error.restype = ctypes.c_char_p
    lib.gf_abi_version.restype = ctypes.c_int
    lib.gf_launch_count.restype = ctypes.c_int64
    lib.gf_launch_count.argtypes = []
    lib.gf_host_exp.argtypes = [P, P, ctypes.c_int64]
    lib.gf_host_hypot.argtypes = [P, P, P, ctypes.c_int64]
    lib.gf_host_pairwise_sum.restype = ctypes.c_double
    lib.gf_host_atan2.argtypes = [P, P, P, ctypes.c_int64]
    lib.gf_host_tanh.argtypes = [P, P, ctypes.c_int64]
    lib.gf_host_sincos.argtypes = [P, P, P, ctypes.c_int64]
    lib.gf_npmath_eval.argtypes = [ctypes.c_int32, ctypes.c_int64, P, P, P, P]
    lib.gf_coherence_fill_workspace_bytes.restype = ctypes.c_size_t
    lib.gf_coherence_fill_workspace_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32,
                                                      ctypes.c_int32, ctypes.c_int64]
    lib.gf_coherence_fill.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P, P,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int64, P, P, P, ctypes.c_int32, P, P,
                                      ctypes.c_size_t, P]
    lib.gf_host_pairwise_sum.argtypes = [P, ctypes.c_int32]
    _lib = lib
    return lib


def launch_count() -> int:
    """Kernels this library has launched in the process (gf_launch_count)."""
    return int(load().gf_launch_count())


def check(rc: int) -> None:
    if rc != GF_OK:
        msg = load().gf_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise NativeError(f"gf error {rc}: {msg}")


def require_cuda():
    """The CUDA device the engine runs on; raise loudly when there is none."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1611_05319_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())
