"""ctypes binding of libtdb200.so (include/td_api.h).

The product path has no CPU fallback: every call here goes to the sm_100a
kernels, and a missing library or GPU raises immediately.  numpy structured
dtypes below mirror the C structs byte for byte (sizes asserted at import).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TD_LIB", os.path.join(HERE, "libtdb200.so"))  # TD_LIB: tuning experiments

# enums (td_api.h)
F32, BF16, F16, F64 = 0, 1, 2, 3
FMT_NONE, FMT_FP32, FMT_BF16, FMT_FP8E4M3 = 0, 1, 2, 3
PASS, FLAG, REPLICA, MERGE, MISSING = 0, 1, 2, 3, 4
GEN_SPLITMIX64, GEN_PHILOX4x32 = 0, 1
MAX_Z = 7
PARTIAL_STRIDE = 10
WARPS_PER_TILE = 8
TILE_UNITS = int(os.environ.get("TD_TILE_UNITS", "8192"))  # must match the library build
SLOT_STRIDE = 8
SEG_HAS_X = 1
SEG_VEC = 2
SEG_TILE_SHIFT_POS = 8
REL_ERR_WORK_BYTES = 16 * 1024 + 16   # TD_REL_ERR_WORK_BYTES
FP_CHUNK = 1 << 18          # bytes per td_fingerprint work chunk (TD_FP_CHUNK)
FP_ITEM = np.dtype([("ptr", "<u8"), ("nbytes", "<i8")])

SEGMENT = np.dtype([
    ("x", "<u8"), ("y", "<u8"), ("z", "<u8", (MAX_Z,)),
    ("x_stride", "<i8"), ("y_stride", "<i8"), ("rows", "<i8"), ("cols", "<i8"),
    ("tile_begin", "<i8"), ("n_units", "<i8"),
    ("x_dtype", "<i4"), ("y_dtype", "<i4"), ("nz", "<i4"), ("flags", "<u4"),
    ("div_m", "<u4"), ("div_p", "<i4"),
    ("y_word0", "<i8"), ("digest_slot", "<i4"), ("pad", "<i4"),
])
ID_DESC = np.dtype([
    ("tile_begin", "<i8"), ("tile_end", "<i8"),
    ("cgroup_begin", "<i4"), ("cgroup_end", "<i4"),
    ("rgroup_begin", "<i4"), ("rgroup_end", "<i4"),
    ("has_compare", "<i4"), ("cand_host", "<i4"), ("ref_host", "<i4"), ("pad", "<i4"),
    ("tolerance", "<f8"),
])
GROUP_DESC = np.dtype([("tile_begin", "<i8"), ("tile_end", "<i8"), ("nz", "<i4"), ("pad", "<i4")])
ID_RESULT = np.dtype([("observed", "<f8"), ("threshold", "<f8"), ("verdict", "<i4"),
                      ("cand_kind", "<i4"), ("ref_kind", "<i4"), ("near_tie", "<i4")])
GROUP_RESULT = np.dtype([("worst", "<f8"), ("worst_index", "<i4"), ("mismatch", "<i4")])
CHUNK = np.dtype([("row_begin", "<i8"), ("row_end", "<i8"), ("k0", "<i4"), ("nk", "<i4")])
assert CHUNK.itemsize == 24
CLASS = np.dtype([("tiles", "<u8"), ("n_tiles", "<i8"), ("dtype", "<i4"), ("nz", "<i4"),
                  ("has_x", "<i4"), ("vec", "<i4"), ("mode", "<i4"), ("digest", "<i4"),
                  ("atol", "<f8"), ("rtol", "<f8"), ("digests", "<u8"), ("host_seg", "<u8")])
MODE_NORMS, MODE_STATIC = 0, 1

assert SEGMENT.itemsize == 160 and ID_DESC.itemsize == 56 and GROUP_DESC.itemsize == 24
assert ID_RESULT.itemsize == 32 and GROUP_RESULT.itemsize == 16 and CLASS.itemsize == 72

# every function the header declares, with its ctypes signature
_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_D = ctypes.c_double
SIGNATURES = {
    "td_version": (ctypes.c_int, []),
    "td_last_error": (ctypes.c_char_p, []),
    "td_sm_count": (ctypes.c_int, [ctypes.c_int]),
    "td_segnorm": (ctypes.c_int, [_P, _P, _I32, _P, _I32, _P]),
    "td_reduce_slots": (ctypes.c_int, [_P, _I32, _P, _I32, _P, _P, _P, _P]),
    "td_verdict": (ctypes.c_int, [_P, _I32, _P, _I32, _P, _P, _D, _D, _D, _P, _P, _P, _P]),
    "td_reduce_chunks": (ctypes.c_int, [_P, _P, _I64, _P, _P]),
    "td_finalize": (ctypes.c_int, [_P, _I32, _P, _I32, _P, _P, _P, _D, _D, _D, _P, _P, _P, _P]),
    "td_perturb": (ctypes.c_int, [_P, _P, _I32, _I32, _I64, _I64, _I64, _I64, _P, _I64, _U64, _D,
                                  _I32, _I32, _P, _P]),
    "td_signed_uniforms": (ctypes.c_int, [_P, _I64, _U64, _I64, _I32, _P]),
    "td_quantize": (ctypes.c_int, [_P, _P, _I32, _I64, _I32, _P, _P]),
    "td_fingerprint": (ctypes.c_int, [_P, _P, _I32, _I64, _P, _P]),
    "td_rel_err": (ctypes.c_int, [_P, _P, _I32, _I64, _P, _P, _P]),
    "td_allreduce_partials": (ctypes.c_int, [_P, _P, _I64, _P]),
    "td_allreduce_digests": (ctypes.c_int, [_P, _P, _I64, _P]),
    "td_allgather_exchange": (ctypes.c_int, [_P, _P, _P, _I64, _P]),
    "td_combine": (ctypes.c_int, [_P, _I32, _I64, _I64, _P, _P, _P, _I64, _P, _P, _P]),
    "td_box_gather": (ctypes.c_int, [_P, _I32, _P, _P, _I32, _P]),
    "td_gather_bytes": (ctypes.c_int, [_P, _P, _P, _I64, _P]),
    "td_generate": (ctypes.c_int, [_P, _I64, _U64, _I32, _D, _D, _I64, _P, _I32, _P, _P, _I32, _P]),
}

_lib = None


class NativeError(RuntimeError):
    """The CUDA extension is missing, failed to load, or a kernel call failed."""


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load and type the library without touching the GPU (works on CPU hosts)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeError(
            f"{path} is missing: build it with `python -m paper_2506_09280_b200.build` "
            "(there is no CPU fallback for the compare path)")
    import torch  # noqa: F401  -- make torch's CUDA runtime resident first
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_HOST_EXT = None


def host_ext():
    """The warm-check record walks in C++ (csrc/td_host.cpp, built in-tree by
    build.build_host), or None: they are host metadata walks with a Python
    twin, so a missing or disabled (TD_HOST_EXT=0) module only costs time."""
    global _HOST_EXT
    if _HOST_EXT is None:
        mod = False
        if os.environ.get("TD_HOST_EXT", "1") != "0":
            try:
                import torch  # noqa: F401  -- libtorch_python resident first
                from . import _td_host as mod
            except ImportError:
                mod = False
        _HOST_EXT = mod
    return _HOST_EXT or None


def lib() -> ctypes.CDLL:
    """The library, on a machine that can actually run it."""
    import torch
    library = load_library()
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the B200 compare path cannot run here")
    return library


def call(name: str, *args) -> None:
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = _lib.td_last_error().decode("utf-8", "replace")
        raise NativeError(f"{name} failed: {msg}")


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


_TORCH_CODES = None


def dtype_code(t) -> int:
    """td_dtype of a torch tensor or numpy array."""
    global _TORCH_CODES
    import torch
    if _TORCH_CODES is None:
        _TORCH_CODES = {torch.float32: F32, torch.bfloat16: BF16, torch.float16: F16,
                        torch.float64: F64}
    if isinstance(t, torch.Tensor):
        code = _TORCH_CODES.get(t.dtype)
    else:
        code = {np.dtype(np.float32): F32, np.dtype(np.float16): F16,
                np.dtype(np.float64): F64}.get(np.asarray(t).dtype)
    if code is None:
        raise TypeError(f"unsupported payload dtype {getattr(t, 'dtype', type(t))}")
    return code


DTYPE_SIZE = {F32: 4, BF16: 2, F16: 2, F64: 8}
