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

from .perturb import PerturbSpec, apply_perturbation
from .torchtap import TapConfig, attach, detach
from .torchtap.writer import encode_id


def torch_runner(model, step: Callable, *, embedding: str, tap: TapConfig,
                 module_inputs: tuple = (), policy: str = "bf16",
                 generator: str = "splitmix64", header: dict | None = None) -> Callable:
    """runner(spec) for estimate_tolerance.

    model:     the torch module (already on the GPU)
    step:      step(model) runs one forward + backward
    embedding: torch name of the module whose output is perturbed
    tap:       which modules to trace and how to name them
    module_inputs: torch names whose first input is perturbed too (module-wise)
    """
    emb = model.get_submodule(embedding)
    emb_id = encode_id(tap.iteration, tap.microbatch, "ActivationOut", tap.canonical_name(embedding))

    def runner(spec: PerturbSpec | None):
        hooks = []
        if spec is not None and spec.eps != 0.0:
            def out_hook(module, args, output):
                return apply_perturbation(output, emb_id, spec, policy=policy, generator=generator)
            hooks.append(emb.register_forward_hook(out_hook, prepend=True))
            for name in module_inputs:
                ident = encode_id(tap.iteration, tap.microbatch, "ActivationIn", tap.canonical_name(name))

                def pre_hook(module, args, _ident=ident):
                    if not args:
                        return None
                    return (apply_perturbation(args[0], _ident, spec, policy=policy,
                                               generator=generator),) + tuple(args[1:])
                hooks.append(model.get_submodule(name).register_forward_pre_hook(pre_hook, prepend=True))
        handle = attach(model, tap)
        try:
            model.zero_grad(set_to_none=True)
            step(model)
        finally:
            detach(handle)
            for h in hooks:
                h.remove()
        hdr = header if header is not None else dict(handle.header(), mode="module-wise" if module_inputs else "cascade")
        return handle.trace(hdr)
    return runner
