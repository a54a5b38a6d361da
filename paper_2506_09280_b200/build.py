"""Build the in-tree C-ABI shared library (libtdb200.so) for sm_100a.

    python -m paper_2506_09280_b200.build

nvcc cross-compiles without a GPU; the .so lands next to this file so it
travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "td_kernels.cu")]
INCLUDE = os.path.join(ROOT, "include")
OUTPUT = os.path.join(HERE, "libtdb200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libtdb200.so")


def needs_build() -> bool:
    if not os.path.exists(OUTPUT):
        return True
    out_m = os.path.getmtime(OUTPUT)
    deps = SOURCES + [os.path.join(INCLUDE, "td_api.h"), __file__]
    return any(os.path.getmtime(p) > out_m for p in deps)


HOST_SOURCE = os.path.join(HERE, "csrc", "td_host.cpp")


def host_output() -> str:
    import sysconfig
    return os.path.join(HERE, "_td_host" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_host(force: bool = False, verbose: bool = False) -> str:
    """The warm-check record walks (csrc/td_host.cpp) as a CPython extension
    against the installed torch (host code only, g++)."""
    import sysconfig

    import torch
    from torch.utils import cpp_extension
    out = host_output()
    if not force and os.path.exists(out) and os.path.getmtime(out) > max(
            os.path.getmtime(HOST_SOURCE), os.path.getmtime(__file__)):
        return out
    libdirs = cpp_extension.library_paths()
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-shared", "-fPIC", "-w",
           f"-D_GLIBCXX_USE_CXX11_ABI={int(torch._C._GLIBCXX_USE_CXX11_ABI)}",
           "-I", sysconfig.get_paths()["include"],
           *[f for d in cpp_extension.include_paths() for f in ("-I", d)],
           HOST_SOURCE, "-o", out + ".tmp",
           *[f"-L{d}" for d in libdirs], *[f"-Wl,-rpath,{d}" for d in libdirs],
           "-lc10", "-ltorch", "-ltorch_cpu", "-ltorch_python"]
    if verbose:
        print(" ".join(cmd), flush=True)
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"g++ failed ({proc.returncode}):\n{proc.stderr}")
    os.replace(out + ".tmp", out)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    try:
        build_host(force=force, verbose=verbose)
    except Exception as exc:       # optional module: the Python walks stand in for it
        print(f"warning: _td_host not built ({exc}); the Python record walks will be used", file=sys.stderr)
    if not force and not needs_build():
        return OUTPUT
    tmp = OUTPUT + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, "-I", INCLUDE, "-o", tmp, *SOURCES]
    if verbose:
        print(" ".join(cmd), flush=True)
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{proc.stderr}")
    if verbose and proc.stderr.strip():
        print(proc.stderr, file=sys.stderr)
    os.replace(tmp, OUTPUT)
    return OUTPUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
