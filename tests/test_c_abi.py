"""The C ABI from a C host (no Python, no torch): tests/c_abi/abi_smoke.c is
compiled with gcc against include/td_api.h and linked to libtdb200.so and
the CUDA runtime — the binding a cgo / JNI / N-API maintainer would write.
Compiling runs on CPU; running it needs the GPU."""

import os
import shutil
import subprocess

import pytest

from paper_2506_09280_b200 import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c_abi", "abi_smoke.c")
CUDA = "/usr/local/cuda"


def _compile(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None or not os.path.exists(os.path.join(CUDA, "include", "cuda_runtime.h")):
        pytest.skip("no C compiler or CUDA headers")
    lib_dir = os.path.dirname(build.OUTPUT)
    if not os.path.exists(build.OUTPUT):
        pytest.skip("libtdb200.so not built")
    exe = tmp_path / "abi_smoke"
    subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-I", build.INCLUDE, "-I", os.path.join(CUDA, "include"),
                    "-o", str(exe), SRC, "-L", lib_dir, "-l:libtdb200.so", "-L", os.path.join(CUDA, "lib64"),
                    "-lcudart", "-lm", "-ldl", f"-Wl,-rpath,{lib_dir}:{os.path.join(CUDA, 'lib64')}"], check=True)
    return exe


def test_c_host_compiles_against_the_header(tmp_path):
    assert _compile(tmp_path).exists()


@pytest.mark.gpu
def test_c_host_runs_on_the_gpu(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _compile(tmp_path)
    proc = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert proc.returncode == 0, proc.stderr
    assert "c abi ok" in proc.stdout and "nccl exchange checked" in proc.stdout, proc.stdout
