"""Runners for estimate_tolerance on a real PyTorch model.

The reference replays its numpy emulator under a PerturbSpec
(checker.py:46, engine.py:1099-1128).  On B200 the trusted model runs for
real: `torch_runner` returns runner(spec) -> Trace that replays one training
step with device-resident torchtap hooks attached and, when spec is given,
the td_perturb kernel applied to the embedding output (cascade mode,
engine.py:466-471) or to every listed module input (module-wise mode,
engine.py:363-386) — the perturbed tensor is what the hooks record, as in
the reference.  Forward/backward stay on PyTorch/cuBLAS.
"""

from __future__ import annotations

from typing import Callable

import torch

from .errors import NonFinite
from .perturb import PerturbSpec, apply_perturbation, straight_through
from .torchtap import TapConfig, attach, detach
from .torchtap.writer import encode_id


def torch_runner(model, step: Callable, *, embedding: str, tap: TapConfig,
                 module_inputs: tuple = (), rewrite: bool = False, rewrite_std: float = 0.02,
                 policy: str = "bf16", generator: str = "splitmix64",
                 header: dict | None = None) -> Callable:
    """runner(spec) for estimate_tolerance.

    model:     the torch module (already on the GPU)
    step:      step(model) runs one forward + backward
    embedding: torch name of the module whose output is perturbed
    tap:       which modules to trace and how to name them
    module_inputs: torch names whose first input is perturbed too (module-wise)
    rewrite:   module-wise mode proper (engine.py:363-377): each listed
               module's input is first REGENERATED from its canonical id —
               generate_full(ActivationIn id, Normal(0, rewrite_std)) on the
               GPU, rounded to the storage format — so every module sees a
               fixed input and only its own perturbation, then perturbed
    """
    emb = model.get_submodule(embedding)
    emb_id = encode_id(tap.iteration, tap.microbatch, "ActivationOut", tap.canonical_name(embedding))

    def runner(spec: PerturbSpec | None, sink=None):
        """One traced step.  With sink, captures stream to sink(ident,
        tensor, module_class) and nothing is kept (returns None)."""
        hooks = []
        # one device counter of non-finite perturbed values per step, read
        # once after it (no host sync inside the forward pass)
        nonfinite = torch.zeros(1, dtype=torch.int64, device="cuda")
        if rewrite:
            for name in module_inputs:
                ident = encode_id(tap.iteration, tap.microbatch, "ActivationIn", tap.canonical_name(name))

                def regen(module, args, _ident=ident):
                    if not args:
                        return None
                    x = args[0]
                    value = _regenerate(_ident, tuple(x.shape), rewrite_std, policy).to(x.dtype)
                    if spec is not None and spec.eps != 0.0:
                        value = apply_perturbation(value, _ident, spec, policy=policy, generator=generator,
                                                   check=False, nonfinite=nonfinite)
                    # the module reads `value`; its input gradient still flows
                    # back to the chain unchanged (engine.py:383-385)
                    return (straight_through(x, value),) + tuple(args[1:])
                hooks.append(model.get_submodule(name).register_forward_pre_hook(regen, prepend=True))
        if spec is not None and spec.eps != 0.0:
            def out_hook(module, args, output):
                # the nudged output replaces the live one; gradients pass
                # through unchanged (straight_through)
                return straight_through(output, apply_perturbation(output, emb_id, spec, policy=policy,
                                                                   generator=generator, check=False,
                                                                   nonfinite=nonfinite))
            hooks.append(emb.register_forward_hook(out_hook, prepend=True))
            for name in (() if rewrite else module_inputs):
                ident = encode_id(tap.iteration, tap.microbatch, "ActivationIn", tap.canonical_name(name))

                def pre_hook(module, args, _ident=ident):
                    if not args:
                        return None
                    return (straight_through(args[0], apply_perturbation(args[0], _ident, spec, policy=policy,
                                                                         generator=generator, check=False,
                                                                         nonfinite=nonfinite)),) + tuple(args[1:])
                hooks.append(model.get_submodule(name).register_forward_pre_hook(pre_hook, prepend=True))
        handle = attach(model, tap, sink=sink)
        try:
            model.zero_grad(set_to_none=True)
            step(model)
        finally:
            detach(handle)
            for h in hooks:
                h.remove()
        if spec is not None and spec.eps != 0.0 and int(nonfinite.item()):
            raise NonFinite("non-finite values in a perturbed input")
        if sink is not None:
            return None
        hdr = header if header is not None else dict(handle.header(), mode="module-wise" if module_inputs else "cascade")
        return handle.trace(hdr)
    return runner


def _regenerate(ident: str, shape: tuple, std: float, policy: str):
    """generate_full(ident, Normal(0, std), shape) on the GPU, quantised to the
    storage format with the reference's RNE (tensor.py:64-77) — fp64 result."""
    from .canonical import parse_canonical
    from .generation import GenSpec, Normal, generate_full_device
    from .tensor import FloatFormat, quantize_array
    full = generate_full_device(parse_canonical(ident), GenSpec(Normal(0.0, std), shape))
    if policy == "fp32":
        return full
    return quantize_array(full, FloatFormat.BF16)
