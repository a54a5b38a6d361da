"""Real-TP shard annotations for live captures.

`layout_shard(layout, dp=, tp=, cp=)` returns the `TapConfig.shard`
callable of one rank of a Megatron-style run whose geometry `layout`
(layout.Layout) describes: every capture of that rank is tagged with the
ShardMapping, RankMeta 6-tuple and declared replica group size the
reference emulator emits for the same (kind, module) on the same rank
(`_hidden_mapping` / `_logits_mapping` / `_param_mapping`,
pkg/src/traindiff/engine.py:268-296; replica rules at the `_emit` sites
listed in layout.py).  The captured tensors stay on the device, so a live
tensor-parallel run feeds check() / check_distributed() with no host round
trip — where the reference adapter only ever writes identity maps
(pkg/adapter/src/torchtap/writer.py:82).

Captures the layout does not name (the ActivationIn/Out of a block's own
sub-modules, e.g. `model.layers.3.attn.norm`, when a pattern matches them)
are hidden-state tensors inside the block's TP region: they get the block's
hidden map and replica size when their local shape is the hidden shard's,
and anything else raises TapError so a wrong annotation never reaches the
checker.
"""

from __future__ import annotations

from ..layout import Layout
from .errors import TapError


def layout_shard(layout: Layout, *, dp: int = 0, tp: int = 0, cp: int = 0):
    """TapConfig.shard for rank (dp, tp, cp) of `layout`:
    (canonical module name, kind, tensor) -> (ShardMapping, rank, replica)."""
    p = layout.p
    if not (0 <= dp < p.dp and 0 <= tp < p.tp and 0 <= cp < p.cp):
        raise TapError(f"rank dp={dp} tp={tp} cp={cp} is outside the layout "
                       f"(dp={p.dp} tp={p.tp} cp={p.cp})")
    table: dict = {}
    for spec in layout.records():
        r = spec.rank
        if r[0] != dp or r[1] != tp or r[4] != cp:
            continue
        module = spec.ident.split("|mod=", 1)[1]
        # a map does not depend on the microbatch: the first one seen wins
        table.setdefault((spec.kind, module), (spec.mapping, r, spec.replica))
    hidden_rep = 1 if p.sp else p.tp
    hidden = layout.hidden(cp, tp, True)

    def shard(name: str, kind: str, tensor):
        shape = tuple(tensor.shape)
        hit = table.get((kind, name))
        if hit is None and kind in ("ActivationIn", "ActivationOut"):
            owner = _block_of(name)
            if owner is not None and shape == hidden.local_shape:
                pp_r, vp_r = layout.placement(owner)
                hit = (hidden, (dp, tp, pp_r, vp_r, cp, int(p.sp)), hidden_rep)
        if hit is None:
            raise TapError(f"layout has no {kind} map for {name!r} on rank dp={dp} tp={tp} cp={cp}")
        mapping = hit[0]
        if shape != mapping.local_shape:
            raise TapError(f"{kind} capture of {name!r} has shape {shape}, the layout's "
                           f"shard on rank dp={dp} tp={tp} cp={cp} is {mapping.local_shape}")
        return hit

    return shard


def _block_of(name: str):
    """'model.layers.3.attn.norm' -> 'model.layers.3.attn' (sub-module of a block)."""
    parts = name.split(".")
    if len(parts) > 4 and parts[0] == "model" and parts[1] == "layers" and parts[3] in ("attn", "mlp"):
        return ".".join(parts[:4])
    return None
