"""The C-ABI library builds for sm_100a, loads without a GPU and exports
every function include/td_api.h declares (no compute calls here)."""

import os
import re
import subprocess

import pytest

from paper_2506_09280_b200 import _native as N
from paper_2506_09280_b200 import build

HEADER = os.path.join(os.path.dirname(N.HERE), "include", "td_api.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(td_[a-z_0-9]+)\s*\(", text)))


def test_library_builds_and_loads():
    path = build.build()
    assert os.path.exists(path)
    lib = N.load_library()
    assert lib.td_version() == 2


def test_every_declared_symbol_is_exported_and_typed():
    lib = N.load_library()
    declared = _declared()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} lacks a ctypes signature"
    assert set(N.SIGNATURES) == set(declared)


def test_exports_are_extern_c():
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("nm unavailable")
    exported = set(re.findall(r"\bT (td_[a-z_0-9]+)\b", out.stdout))
    assert set(_declared()) <= exported


def test_cubin_is_sm_100a():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_last_error_reports_bad_arguments():
    lib = N.load_library()
    # argument validation happens before any CUDA call, so this is CPU-safe
    rc = lib.td_verdict(None, 5, None, 0, None, None, 3.0, 0.1, 0.1, None, None, None, None)
    assert rc != 0
    assert b"td_verdict" in lib.td_last_error()


def test_struct_layouts_match_header(tmp_path):
    """The numpy mirrors of the ABI structs have the sizes and field offsets
    the C compiler gives include/td_api.h."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {"td_segment": N.SEGMENT, "td_id_desc": N.ID_DESC, "td_group_desc": N.GROUP_DESC,
               "td_id_result": N.ID_RESULT, "td_group_result": N.GROUP_RESULT, "td_class": N.CLASS,
               "td_chunk": N.CHUNK, "td_fp_item": N.FP_ITEM}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "td_api.h"', "int main(void) {"]
    for name, dt in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for field in dt.names:
            lines.append(f'printf("{name}.{field} %zu\\n", offsetof({name}, {field}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", build.INCLUDE, "-o", str(exe), str(src)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for name, dt in structs.items():
        assert int(got[name]) == dt.itemsize, name
        for field in dt.names:
            assert int(got[f"{name}.{field}"]) == dt.fields[field][1], f"{name}.{field}"


def test_integration_stub_matches_the_abi():
    """The ctypes stub a maintainer would paste declares
    the same argument types the library is loaded with (_native.SIGNATURES)."""
    import ctypes
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "INTEGRATION.md")).read()
    kinds = {"_P": ctypes.c_void_p, "_I32": ctypes.c_int32, "_I64": ctypes.c_int64,
             "_U64": ctypes.c_uint64, "_D": ctypes.c_double}
    found = re.findall(r"_lib\.(td_\w+)\.argtypes\s*=\s*\[([^\]]*)\]", text)
    assert len(found) >= 6
    for name, args in found:
        assert [kinds[a.strip()] for a in args.split(",") if a.strip()] == N.SIGNATURES[name][1], name
