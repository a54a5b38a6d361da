"""eps-scaled input perturbation for the tolerance proxy — kernel 2.

Reference: Emulator._perturb_tag / _apply_perturbation
(pkg/src/traindiff/engine.py:348-361): for sample s and tensor id I,

    u      = signed_uniforms("perturb|s={s}|{I}", (seq_len, d_model))
    y[r,:] = Q_fmt(x[r,:] * (1 + u[pos(r), :] * eps))

where pos(r) is the global sequence position of local row r (zigzag CP /
SP sub-slices, engine.py:148-168) and Q_fmt is the storage quantiser
(tensor.py:64-77; identity for the fp32 policy).  td_perturb fuses stream
generation, the fp64 arithmetic (each op rounded on its own, like numpy)
and the cast into one pass over the rank's own rows.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native as N
from .canonical import CanonicalId
from .errors import NonFinite
from .generation import GENERATORS, seed_from


@dataclass(frozen=True)
class PerturbSpec:
    """x -> x * (1 + u*eps), u ~ U[-1, 1] keyed by (sample, tensor id)
    (engine.py:187-192)."""

    sample: int
    eps: float


def perturb_tag(spec: PerturbSpec, ident) -> str:
    text = ident.encode() if isinstance(ident, CanonicalId) else str(ident)
    return f"perturb|s={spec.sample}|{text}"


_FMT_BY_POLICY = {"fp32": N.FMT_NONE, "bf16": N.FMT_BF16, "bf16-fp8": N.FMT_BF16}


def apply_perturbation(x, ident, spec: PerturbSpec | None, *, full_cols: int | None = None,
                       row_positions=None, row0: int = 0, col0: int = 0,
                       policy: str = "fp32", fmt: int | None = None,
                       out=None, generator: str = "splitmix64", check: bool = True,
                       nonfinite=None):
    """Perturbed copy of the CUDA tensor x (rows, cols) — or x itself when
    spec is None or spec.eps == 0 (engine.py:355-356).

    full_cols: width of the full logical tensor (d_model); defaults to x's.
    row_positions: global row of each local row (CUDA/host int64), or rows
    are row0, row0+1, ....  fmt overrides the policy's storage quantiser.
    check=False leaves the non-finite test to the caller, who passes a
    `nonfinite` device counter and inspects it later (no host sync)."""
    import torch
    if spec is None or spec.eps == 0.0:
        return x
    if x.dim() == 1:
        rows, cols = 1, x.shape[0]
    else:
        cols = x.shape[-1]
        rows = x.numel() // max(cols, 1)
    full = cols if full_cols is None else int(full_cols)
    src = x if x.is_contiguous() else x.contiguous()
    y = torch.empty_like(src) if out is None else out
    pos = None
    if row_positions is not None:
        pos = torch.as_tensor(row_positions, dtype=torch.int64, device=src.device)
    counter = nonfinite if nonfinite is not None else torch.zeros(1, dtype=torch.int64, device=src.device)
    code = _FMT_BY_POLICY[policy] if fmt is None else fmt
    N.call("td_perturb", src.data_ptr(), y.data_ptr(), N.dtype_code(src), N.dtype_code(y),
           rows, cols, full, col0, pos.data_ptr() if pos is not None else None, row0,
           seed_from(perturb_tag(spec, ident)), float(spec.eps), code, GENERATORS[generator],
           counter.data_ptr(), N.stream_handle())
    if check and nonfinite is None and int(counter.item()) != 0:
        raise NonFinite("non-finite values in perturbed input")
    return y


_STRAIGHT = None


def straight_through(x, value):
    """`value` in the forward pass, the gradient handed to `x` unchanged in
    the backward: how a perturbed (or regenerated) tensor stands in for a
    live activation.  The reference's backward uses the gradient of the
    module's output as is for the upstream chain and the embedding's
    parameters (engine.py:886-908, 383-385) — the (1 + u*eps) factor is an
    input nudge, not part of the differentiated function.  A plain
    td_perturb output has no autograd history, so returning it from a hook
    would cut the graph: no gradient would reach anything upstream."""
    global _STRAIGHT
    import torch
    if not (torch.is_grad_enabled() and x.requires_grad):
        return value
    if _STRAIGHT is None:
        class StraightThrough(torch.autograd.Function):
            @staticmethod
            def forward(ctx, inp, val):
                return val.clone()

            @staticmethod
            def backward(ctx, grad):
                return grad, None
        _STRAIGHT = StraightThrough.apply
    return _STRAIGHT(x, value)


def perturb_hook(ident, spec: PerturbSpec | None, *, policy: str = "fp32", row_positions=None,
                 generator: str = "splitmix64"):
    """A torch forward hook that replaces a module's output with its
    perturbed version — how the B200 runner applies the proxy to the
    embedding output (engine.py:466-471)."""
    def hook(module, args, output):
        if spec is None or spec.eps == 0.0:
            return output
        return straight_through(output, apply_perturbation(output, ident, spec, policy=policy,
                                                           row_positions=row_positions, generator=generator))
    return hook


def perturb_pre_hook(ident, spec: PerturbSpec | None, *, policy: str = "fp32", row_positions=None,
                     generator: str = "splitmix64"):
    """Forward-pre hook perturbing a module's first input (module-wise mode,
    engine.py:363-386)."""
    def hook(module, args):
        if spec is None or spec.eps == 0.0 or not args:
            return None
        first = apply_perturbation(args[0], ident, spec, policy=policy,
                                   row_positions=row_positions, generator=generator)
        return (straight_through(args[0], first),) + tuple(args[1:])
    return hook
