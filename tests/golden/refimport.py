"""Import the read-only reference package (only in the build container).

Used by make_golden.py and by the reference-pinning CPU tests; nothing on the
GPU box imports this (the reference tree does not exist there).
"""
import os
import sys

REF_SRC = "/root/reference/pkg/src"
_STUB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_refstub")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "guidefill"))


def load():
    if not available():
        raise ImportError("reference package not present")
    # tests/ref_suite binds the name guidefill to paper_1611_05319_b200: drop
    # that alias before importing the real reference
    mod = sys.modules.get("guidefill")
    if mod is not None and not str(getattr(mod, "__file__", "")).startswith(REF_SRC):
        for name in [k for k in sys.modules if k == "guidefill" or k.startswith("guidefill.")]:
            del sys.modules[name]
    for p in (_STUB, REF_SRC):
        if p not in sys.path:
            sys.path.insert(0, p)
    import guidefill  # noqa: F401
    from guidefill import engine, grid, guide, splines, tracker
    return dict(engine=engine, grid=grid, guide=guide, splines=splines, tracker=tracker,
                guidefill=guidefill)
