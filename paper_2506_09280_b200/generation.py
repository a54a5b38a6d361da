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
