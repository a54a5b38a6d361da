"""Counter-based random streams (drop-in for the perturbation half of
pkg/src/traindiff/generation.py).

The seed of a stream is FNV-1a-64 of a tag string (generation.py:36-46);
word k of the stream is splitmix64's output for state seed + (k+1)*gamma
(generation.py:49-78).  Because word k depends on k alone, each rank
generates exactly the slice it owns on the GPU (td_signed_uniforms,
td_perturb) with no communication.  Philox4x32-10 is offered as an opt-in
generator (`generator="philox"`); its CPU restatement lives in the tests.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .canonical import CanonicalId

_FNV_OFFSET = 0xCBF29CE484222325
_FNV_PRIME = 0x100000001B3
_M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB

GENERATORS = {"splitmix64": N.GEN_SPLITMIX64, "philox": N.GEN_PHILOX4x32}


def fnv1a_64(data: bytes) -> int:
    h = _FNV_OFFSET
    for byte in data:
        h = ((h ^ byte) * _FNV_PRIME) & _M64
    return h


def seed_from(ident) -> int:
    """Seed of a tensor's private stream: FNV-1a of its canonical id / tag."""
    text = ident.encode() if isinstance(ident, CanonicalId) else ident
    return fnv1a_64(text.encode("utf-8"))


class SplitMix64:
    """Scalar stream stepping, the semantics the device generator reproduces."""

    def __init__(self, seed: int):
        self._state = seed & _M64

    def next_word(self) -> int:
        self._state = (self._state + GAMMA) & _M64
        z = self._state
        z = ((z ^ (z >> 30)) * MIX1) & _M64
        z = ((z ^ (z >> 27)) * MIX2) & _M64
        return z ^ (z >> 31)

    def next_uniform(self) -> float:
        return (self.next_word() >> 11) * 2.0 ** -53


def signed_uniforms_device(tag_or_seed, n: int, k0: int = 0, generator: str = "splitmix64"):
    """Uniforms 2u-1 in [-1, 1] for counters k0..k0+n-1, as a CUDA f64 tensor."""
    import torch
    seed = tag_or_seed if isinstance(tag_or_seed, int) else seed_from(tag_or_seed)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    N.call("td_signed_uniforms", out.data_ptr(), n, seed & _M64, k0, GENERATORS[generator],
           N.stream_handle())
    return out


def signed_uniforms(tag: str, shape: tuple[int, ...], generator: str = "splitmix64") -> np.ndarray:
    """Reference-shaped host array (generation.py:163-167), generated on the GPU."""
    n = math.prod(shape)
    return signed_uniforms_device(tag, n, 0, generator).cpu().numpy().reshape(shape)


# ---------------------------------------------------------------------------
# generate_full on the device (generation.py:81-186)

@dataclass(frozen=True)
class Normal:
    mean: float = 0.0
    std: float = 1.0


@dataclass(frozen=True)
class Uniform:
    low: float = 0.0
    high: float = 1.0


@dataclass(frozen=True)
class TokenIds:
    vocab: int


@dataclass(frozen=True)
class GenSpec:
    distribution: object
    shape: tuple

    def __post_init__(self):
        object.__setattr__(self, "shape", tuple(int(n) for n in self.shape))
        if any(n <= 0 for n in self.shape):
            raise ValueError(f"non-positive dimension in shape {self.shape}")
        if isinstance(self.distribution, TokenIds) and self.distribution.vocab < 1:
            raise ValueError("token vocabulary must be positive")


def generate_full_device(ident, spec: GenSpec):
    """The full logical tensor for `ident` under `spec`, as a CUDA f64
    tensor (td_generate).  Uniform and token streams are bit-exact with the
    reference; normals use CUDA's log/cos/sin (<= 2 ulp) and so agree to
    ~1e-16 relative (the reference's own normal test allows 1e-15,
    test_generation.py:59-63).  Exact-zero uniforms (2^-53 per word) are
    skipped exactly like the reference's scalar fallback."""
    import torch
    seed = seed_from(ident)
    n = math.prod(spec.shape)
    d = spec.distribution
    if isinstance(d, Normal):
        code, a, b, vocab = 0, float(d.mean), float(d.std), 1
    elif isinstance(d, Uniform):
        code, a, b, vocab = 1, float(d.low), float(d.high), 1
    elif isinstance(d, TokenIds):
        code, a, b, vocab = 2, 0.0, 0.0, int(d.vocab)
    else:
        raise TypeError(f"unknown distribution {d!r}")
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    cap = 64
    count = torch.zeros(1, dtype=torch.int64, device="cuda")
    pos = torch.zeros(cap, dtype=torch.int64, device="cuda")
    skips: list = []
    while True:
        sk = torch.tensor(skips, dtype=torch.int64, device="cuda") if skips else None
        count.zero_()
        N.call("td_generate", out.data_ptr(), n, seed & _M64, code, a, b, vocab,
               sk.data_ptr() if sk is not None else None, len(skips),
               count.data_ptr() if code == 0 else None, pos.data_ptr(), cap, N.stream_handle())
        if code != 0:
            break
        seen = int(count.item())
        if seen > cap:
            raise N.NativeError(f"{seen} zero uniforms in one stream; skip list capacity is {cap}")
        found = sorted(int(p) for p in pos[:seen].cpu().tolist())
        if found == skips:
            break
        skips = found
    return out.reshape(spec.shape)


def generate_full(ident, spec: GenSpec, device=None):
    """Reference-shaped generate_full (generation.py:146-160): a host Tensor,
    or the CUDA tensor itself with device="cuda"."""
    t = generate_full_device(ident, spec)
    if device is not None:
        return t
    from .tensor import Tensor
    return Tensor(t.cpu().numpy())


def extract_shard(full, mapping):
    """The shard a rank holding `mapping` sees of `full` (generation.py:170-186)."""
    from .canonical import validate_mapping
    from .errors import MappingInvalid
    validate_mapping(mapping)
    data = getattr(full, "data", full)
    if tuple(data.shape) != mapping.global_shape:
        raise MappingInvalid(
            f"full tensor shape {tuple(data.shape)} != mapping global shape {mapping.global_shape}")
    if sum(loc.volume for loc, _ in mapping.pairs) != math.prod(mapping.local_shape):
        raise MappingInvalid("local boxes do not cover the local shape")
    import torch
    out = torch.zeros(mapping.local_shape, dtype=data.dtype, device=data.device) \
        if isinstance(data, torch.Tensor) else np.zeros(mapping.local_shape, dtype=np.float64)
    for loc, glob in mapping.pairs:
        out[loc.as_slices()] = data[glob.as_slices()]
    return out
