"""Storage formats and the relative-error primitive (drop-in for
pkg/src/traindiff/tensor.py:28-77,144-167).

`FloatFormat` and `Tensor` are host metadata/containers with the reference's
semantics.  The arithmetic — rel_err_arrays' two fp64 norms and
quantize_array's RNE-to-p-bits — runs in the sm_100a kernels (td_segnorm,
td_quantize).  The reference's emulator arithmetic (PolicyOps, einsum
matmul) is out of scope: on B200 the traced model runs in PyTorch/cuBLAS.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import NonFinite, ShapeMismatch


class FloatFormat(enum.Enum):
    FP32 = "FP32"
    BF16 = "BF16"
    FP8E4M3 = "FP8E4M3"

    @property
    def precision(self) -> int:
        """Significand bits including the implicit one."""
        return {FloatFormat.FP32: 24, FloatFormat.BF16: 8, FloatFormat.FP8E4M3: 4}[self]

    @property
    def eps(self) -> float:
        """Unit roundoff 2**-precision."""
        return 2.0 ** -self.precision

    @property
    def max_finite(self) -> float:
        return {FloatFormat.FP32: float(np.finfo(np.float32).max),
                FloatFormat.BF16: 1.9921875 * 2.0 ** 127,
                FloatFormat.FP8E4M3: 448.0}[self]

    @property
    def code(self) -> int:
        return {FloatFormat.FP32: N.FMT_FP32, FloatFormat.BF16: N.FMT_BF16,
                FloatFormat.FP8E4M3: N.FMT_FP8E4M3}[self]


@dataclass(frozen=True)
class Tensor:
    """A shaped value.  Host data is float64 numpy as in the reference;
    CUDA tensors are kept as they are (device-resident payloads)."""

    data: object

    def __post_init__(self):
        from .device import is_torch
        if not is_torch(self.data):
            object.__setattr__(self, "data", np.asarray(self.data, dtype=np.float64))

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(self.data.shape)

    @classmethod
    def zeros(cls, shape: tuple[int, ...]) -> "Tensor":
        return cls(np.zeros(shape, dtype=np.float64))

    @classmethod
    def full(cls, shape: tuple[int, ...], value: float) -> "Tensor":
        return cls(np.full(shape, value, dtype=np.float64))


def _shape(x) -> tuple[int, ...]:
    return tuple(x.shape) if hasattr(x, "shape") else tuple(np.shape(x))


def rel_err_arrays(a, b) -> float:
    """||a - b||_F / ||a||_F in fp64 on the GPU; 0/0 -> 0.0, x/0 -> +inf
    (tensor.py:158-167).  Accepts numpy arrays or torch tensors (any device)."""
    sa, sb = _shape(a), _shape(b)
    if sa != sb:
        raise ShapeMismatch(f"rel_err: {sa} vs {sb}")
    from .device import rel_err_pair
    return rel_err_pair(a, b)


def rel_err(a: Tensor, b: Tensor) -> float:
    return rel_err_arrays(a.data, b.data)


def frobenius_norm(a: Tensor) -> float:
    """sqrt(sum a^2) (tensor.py:144-145): the reference-norm sum of a
    self-compare (td_rel_err with b = a), reduced on the GPU."""
    from .device import pair_sums, to_device
    ta = to_device(a.data).reshape(-1)
    return float(np.sqrt(pair_sums(ta, ta)[1]))


def quantize_array(x, fmt: FloatFormat) -> np.ndarray:
    """RNE to fmt's significand precision with unbounded exponent, clamped to
    +-max_finite (tensor.py:64-77); td_quantize works on the fp64 bit
    pattern, never through float32.  Returns float64 like the reference."""
    import torch
    from .device import to_device
    from .device import is_torch
    host = not (is_torch(x) and x.device.type == "cuda")
    src = to_device(np.asarray(x.cpu() if is_torch(x) else x, dtype=np.float64) if host
                    else x.to(torch.float64))
    out = torch.empty_like(src)
    flag = torch.zeros(1, dtype=torch.int64, device=src.device)
    N.call("td_quantize", src.data_ptr(), out.data_ptr(), N.F64, src.numel(), fmt.code,
           flag.data_ptr(), N.stream_handle())
    if int(flag.item()) != 0:
        raise NonFinite("quantize input contains NaN or infinity")
    return out.cpu().numpy().reshape(np.shape(x)) if host else out


def quantize(a: Tensor, fmt: FloatFormat) -> Tensor:
    return Tensor(quantize_array(a.data, fmt))


@dataclass(frozen=True)
class PrecisionPolicy:
    """Formats a run stores values in and feeds its matmuls with (tensor.py:174-186)."""

    name: str
    storage: FloatFormat
    matmul_inputs: FloatFormat


POLICIES = {
    "fp32": PrecisionPolicy("fp32", FloatFormat.FP32, FloatFormat.FP32),
    "bf16": PrecisionPolicy("bf16", FloatFormat.BF16, FloatFormat.BF16),
    "bf16-fp8": PrecisionPolicy("bf16-fp8", FloatFormat.BF16, FloatFormat.FP8E4M3),
}
