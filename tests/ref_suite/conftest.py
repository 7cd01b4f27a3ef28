"""The reference's own hot-path test suite, run against this package.

The files next to this one are the reference's tests (pkg/tests/) vendored
unchanged apart from a header.  They import ``guidefill``; here that name is
bound to ``paper_1611_05319_b200`` (package and submodules), so every test
exercises the B200 engine through exactly the API a reference user calls --
the drop-in claim of INTEGRATION.md, checked by the reference's own asserts.
The CLI suite runs too (the reference's commands minus ``serve``), and so do
the project store and HTTP service suites (the callers of
the fill path, ``project.py`` / ``service.py`` of this package routing to the
GPU engine).  All of them need the GPU (marked ``gpu``).
"""

import importlib
import sys

import pytest

import paper_1611_05319_b200 as _pkg

for _name in ("engine", "grid", "guide", "splines", "tracker", "harness", "limits", "fileio",
              "cli", "project", "service"):
    sys.modules[f"guidefill.{_name}"] = importlib.import_module(f"paper_1611_05319_b200.{_name}")
sys.modules["guidefill"] = _pkg


# Reference tests whose exact-equality asserts lie outside this build's
# declared contract (fill order bit-exact, values within 1e-4): strict xfail,
# so they are reported, and a pass would be flagged.
KNOWN = {
    "test_iteration_reads_come_from_snapshot":
        "asserts a float64 fill value exactly (0.9); the device colour path is fp32 "
        "(0.8999999761581421), within the 1e-4 value tolerance",
}


def pytest_collection_modifyitems(config, items):
    for item in items:
        if "ref_suite" in str(item.fspath):
            item.add_marker(pytest.mark.gpu)
            if item.name in KNOWN:
                item.add_marker(pytest.mark.xfail(reason=KNOWN[item.name], strict=True))
