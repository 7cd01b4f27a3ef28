"""The C-ABI library loads and exports every symbol include/*.h declares."""

import ctypes
import os
import re

from paper_1611_05319_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "guidefill_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_bound_api():
    decl = declared_functions()
    assert decl, "no declarations parsed"
    assert set(decl) == set(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.gf_abi_version() == 2


def test_struct_layouts_match_the_header(tmp_path):
    # compile the header with the system C compiler and compare sizes/offsets
    import subprocess
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "guidefill_b200.h"\n'
        'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(gf_fill_params),'
        ' sizeof(gf_frames), sizeof(gf_fill_outputs), offsetof(gf_fill_params, g_fixed),'
        ' offsetof(gf_frames, image), offsetof(gf_fill_outputs, enter)); return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(_native.FillParamsC), ctypes.sizeof(_native.FramesC),
            ctypes.sizeof(_native.FillOutputsC), _native.FillParamsC.g_fixed.offset,
            _native.FramesC.image.offset, _native.FillOutputsC.enter.offset]
    assert got == want


def test_invalid_arguments_are_rejected_without_a_device():
    lib = _native.load()
    fr = _native.FramesC(1, 0, 5, 3, 0, 0, 0, 0, 0)
    pc = _native.FillParamsC()
    assert lib.gf_fill_workspace_bytes(ctypes.byref(fr), ctypes.byref(pc)) == 0
    oc = _native.FillOutputsC()
    rc = lib.gf_fill(ctypes.byref(fr), ctypes.byref(pc), ctypes.byref(oc), None, 0, None)
    assert rc == -1
    assert b"geometry" in lib.gf_last_error()
