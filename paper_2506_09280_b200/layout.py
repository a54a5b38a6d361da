"""Shard index maps and id emission of a parallel layout.

Port of the geometry half of the reference emulator — which ids a layout
traces, on which rank, through which shard mapping and with which declared
replica group size — without its arithmetic:

* sequence geometry: zigzag CP stripes and SP sub-slices
  (pkg/src/traindiff/engine.py:148-184, 260-307)
* TP axes of parameters (engine.py:210-222), PP/VP placement (:309-317,
  canonical.py:71-90)
* the emission order and replica rules of Emulator.run_iteration and its
  _emit call sites (engine.py:321-335, 425-1065)

`emit_records(model, pcfg)` yields RecordSpec rows in the reference's
execution order; tests/test_layout.py checks them against the reference
emulator's traces over the 60-layout grid (tests/golden/layouts.json.gz).
The B200 build uses them to lay out synthetic traces of the named model
shapes (bench.py) and to annotate device captures with real-TP maps.

Extensions beyond the reference's GPT model, for the Llama configs:
`gated_mlp` adds a column-parallel `w3`; `n_kv_heads` gives `wk`/`wv` the
GQA width n_kv*head_dim; `norm_bias=False` drops LayerNorm biases
(RMSNorm); `position_table=False` drops the learned position table.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

from .canonical import ShardMapping, SliceBox, locate_layer
from .errors import ConfigInvalid


@dataclass(frozen=True)
class ModelShape:
    layers: int
    d_model: int
    n_heads: int
    d_ff: int
    seq_len: int
    vocab: int
    n_kv_heads: int | None = None
    gated_mlp: bool = False
    norm_bias: bool = True
    position_table: bool = True

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    @property
    def kv_width(self) -> int:
        return (self.n_kv_heads or self.n_heads) * self.head_dim


@dataclass(frozen=True)
class ParallelConfig:
    dp: int = 1
    tp: int = 1
    pp: int = 1
    vp: int = 1
    cp: int = 1
    sp: bool = False
    microbatches: int = 1

    def world_size(self) -> int:
        return self.dp * self.tp * self.pp * self.cp


def validate_parallel(m: ModelShape, p: ParallelConfig, max_world: int = 8) -> None:
    """engine.py:76-94"""
    if min(p.dp, p.tp, p.pp, p.vp, p.cp, p.microbatches) < 1:
        raise ConfigInvalid("parallel degrees and microbatches must be >= 1")
    if p.world_size() > max_world:
        raise ConfigInvalid(f"world size {p.world_size()} exceeds {max_world}")
    if p.microbatches % p.dp:
        raise ConfigInvalid("microbatches must divide evenly across dp ranks")
    if m.layers % (p.pp * p.vp):
        raise ConfigInvalid("layers must be divisible by pp * vp")
    for name in ("d_model", "d_ff", "n_heads", "vocab"):
        if getattr(m, name) % p.tp:
            raise ConfigInvalid(f"{name} must be divisible by tp")
    if p.cp > 1 and m.seq_len % (2 * p.cp):
        raise ConfigInvalid("seq_len must be divisible by 2*cp when cp > 1")
    if p.sp and (m.seq_len // p.cp) % p.tp:
        raise ConfigInvalid("per-cp-rank sequence must be divisible by tp when sp")


# -- sequence geometry ---------------------------------------------------------

def seq_pieces(seq: int, cp: int, c: int) -> list:
    """(local, global) row intervals of CP rank c: zigzag chunks c and 2cp-1-c."""
    if cp == 1:
        return [((0, seq), (0, seq))]
    ch = seq // (2 * cp)
    return [((0, ch), (c * ch, (c + 1) * ch)),
            ((ch, 2 * ch), ((2 * cp - 1 - c) * ch, (2 * cp - c) * ch))]


def sub_pieces(pieces: list, lo: int, hi: int) -> list:
    """Restrict pieces to local rows [lo, hi) and rebase them to 0."""
    out = []
    for (l0, l1), (g0, _) in pieces:
        a, b = max(l0, lo), min(l1, hi)
        if a < b:
            out.append(((a - lo, b - lo), (g0 + a - l0, g0 + b - l0)))
    return out


def piece_positions(pieces: list) -> list[int]:
    return [g for _, (g0, g1) in pieces for g in range(g0, g1)]


def mapping_from(local_shape: tuple, global_shape: tuple, per_axis: dict) -> ShardMapping:
    """Cartesian product of per-axis interval pieces into box pairs."""
    axes = [per_axis.get(a, [((0, n), (0, global_shape[a]))]) for a, n in enumerate(local_shape)]
    pairs = tuple((SliceBox(tuple(p[0] for p in combo)), SliceBox(tuple(p[1] for p in combo)))
                  for combo in itertools.product(*axes))
    return ShardMapping(tuple(local_shape), tuple(global_shape), pairs)


def param_tp_axis(path: str) -> int | None:
    """engine.py:210-218 (+ w3 for gated MLPs)."""
    if path.endswith(".word"):
        return 0
    if path.endswith((".wq", ".wk", ".wv", ".w1", ".w3")):
        return 1
    if path.endswith((".wo", ".w2")):
        return 0
    return None


def is_norm_param(path: str) -> bool:
    return ".norm." in path or path.startswith("model.final_norm.")


def param_shapes(m: ModelShape) -> list[tuple[str, tuple[int, ...]]]:
    """Parameter registration order (model.py:81-112, plus the extensions)."""
    d, ff = m.d_model, m.d_ff
    out = [("model.embedding.word", (m.vocab, d))]
    if m.position_table:
        out.append(("model.embedding.position", (m.seq_len, d)))
    for layer in range(m.layers):
        attn, mlp = f"model.layers.{layer}.attn", f"model.layers.{layer}.mlp"
        out.append((f"{attn}.norm.weight", (d,)))
        if m.norm_bias:
            out.append((f"{attn}.norm.bias", (d,)))
        out += [(f"{attn}.wq", (d, d)), (f"{attn}.wk", (d, m.kv_width)),
                (f"{attn}.wv", (d, m.kv_width)), (f"{attn}.wo", (d, d)),
                (f"{mlp}.norm.weight", (d,))]
        if m.norm_bias:
            out.append((f"{mlp}.norm.bias", (d,)))
        out.append((f"{mlp}.w1", (d, ff)))
        if m.gated_mlp:
            out.append((f"{mlp}.w3", (d, ff)))
        out.append((f"{mlp}.w2", (ff, d)))
    out.append(("model.final_norm.weight", (d,)))
    if m.norm_bias:
        out.append(("model.final_norm.bias", (d,)))
    return out


@dataclass(frozen=True)
class RecordSpec:
    ident: str                 # canonical id string
    rank: tuple                # (dp, tp, pp, vp, cp, sp)
    mapping: ShardMapping
    replica: int
    module_class: str
    kind: str = field(default="")


class Layout:
    """Geometry of one (model, parallel config) pair."""

    def __init__(self, m: ModelShape, p: ParallelConfig, iteration: int = 0):
        validate_parallel(m, p)
        self.m, self.p, self.iteration = m, p, iteration
        self.ranks = [(c, t) for c in range(p.cp) for t in range(p.tp)]
        self.layers_per_chunk = m.layers // (p.pp * p.vp)
        self.params = param_shapes(m)

    def pieces(self, c: int, t: int, sp_domain: bool) -> list:
        pieces = seq_pieces(self.m.seq_len, self.p.cp, c)
        if sp_domain and self.p.sp:
            sub = self.m.seq_len // self.p.cp // self.p.tp
            pieces = sub_pieces(pieces, t * sub, (t + 1) * sub)
        return pieces

    def hidden(self, c: int, t: int, sp_domain: bool) -> ShardMapping:
        pieces = self.pieces(c, t, sp_domain)
        rows = sum(b - a for (a, b), _ in pieces)
        return mapping_from((rows, self.m.d_model), (self.m.seq_len, self.m.d_model), {0: pieces})

    def ids_map(self, c: int) -> ShardMapping:
        pieces = self.pieces(c, 0, False)
        rows = sum(b - a for (a, b), _ in pieces)
        return mapping_from((rows,), (self.m.seq_len,), {0: pieces})

    def logits(self, c: int, t: int) -> ShardMapping:
        pieces = self.pieces(c, 0, False)
        rows = sum(b - a for (a, b), _ in pieces)
        v = self.m.vocab // self.p.tp
        return mapping_from((rows, v), (self.m.seq_len, self.m.vocab),
                            {0: pieces, 1: [((0, v), (t * v, (t + 1) * v))]})

    def param(self, path: str, shape: tuple, t: int) -> ShardMapping:
        axis = param_tp_axis(path)
        if axis is None:
            box = SliceBox(tuple((0, n) for n in shape))
            return ShardMapping(shape, shape, ((box, box),))
        n = shape[axis] // self.p.tp
        local = tuple(n if a == axis else s for a, s in enumerate(shape))
        return mapping_from(local, shape, {axis: [((0, n), (t * n, (t + 1) * n))]})

    def position_grad(self, c: int, t: int) -> ShardMapping:
        pieces = self.pieces(c, t, self.p.sp)
        rows = sum(b - a for (a, b), _ in pieces)
        return mapping_from((rows, self.m.d_model), (self.m.seq_len, self.m.d_model), {0: pieces})

    def placement(self, module: str) -> tuple[int, int]:
        if module.startswith("model.layers."):
            p, v, _ = locate_layer(int(module.split(".")[2]), self.p.pp, self.p.vp,
                                   self.layers_per_chunk)
            return p, v
        if module.startswith("model.embedding"):
            return 0, 0
        return self.p.pp - 1, self.p.vp - 1

    # -- emission -------------------------------------------------------------

    def _rec(self, dr, c, t, mb, kind, module, cls, mapping, replica, iteration=None):
        pp_r, vp_r = self.placement(module)
        it = self.iteration if iteration is None else iteration
        ident = f"iter={it}|mb={mb}|kind={kind}|mod={module}"
        return RecordSpec(ident, (dr, t, pp_r, vp_r, c, int(self.p.sp)), mapping, replica, cls, kind)

    def _params(self, iteration):
        p = self.p
        for path, shape in self.params:
            sharded = param_tp_axis(path) is not None
            replica = p.dp * p.cp * (1 if sharded else p.tp)
            for dr in range(p.dp):
                for c, t in self.ranks:
                    yield self._rec(dr, c, t, 0, "Param", path, "Param", self.param(path, shape, t),
                                    replica, iteration=iteration)

    def _forward(self, dr, mb):
        p, m = self.p, self.m
        rep = 1 if p.sp else p.tp
        for c, t in self.ranks:
            yield self._rec(dr, c, t, mb, "ActivationIn", "model.embedding", "Embedding",
                            self.ids_map(c), p.tp)
        for c in range(p.cp):
            for t in range(p.tp):
                yield self._rec(dr, c, t, mb, "ActivationOut", "model.embedding", "Embedding",
                                self.hidden(c, t, p.sp), 1 if p.sp else p.tp)
        for layer in range(m.layers):
            for name, cls in ((f"model.layers.{layer}.attn", "AttentionBlock"),
                              (f"model.layers.{layer}.mlp", "MlpBlock")):
                for c, t in self.ranks:
                    yield self._rec(dr, c, t, mb, "ActivationIn", name, cls, self.hidden(c, t, True), rep)
                for c in range(p.cp):
                    for t in range(p.tp):
                        yield self._rec(dr, c, t, mb, "ActivationOut", name, cls,
                                        self.hidden(c, t, True), rep)
        for c, t in self.ranks:
            for kind in ("ActivationIn", "ActivationOut"):
                yield self._rec(dr, c, t, mb, kind, "model.final_norm", "LayerNorm",
                                self.hidden(c, t, True), rep)
        for c in range(p.cp):
            for t in range(p.tp):
                yield self._rec(dr, c, t, mb, "ActivationIn", "model.lm_head", "TiedLMHead",
                                self.hidden(c, t, False), p.tp)
                yield self._rec(dr, c, t, mb, "ActivationOut", "model.lm_head", "TiedLMHead",
                                self.logits(c, t), 1)

    def _backward(self, dr, mb):
        p, m = self.p, self.m
        rep = 1 if p.sp else p.tp
        for c in range(p.cp):
            for t in range(p.tp):
                yield self._rec(dr, c, t, mb, "ActivationGradOut", "model.lm_head", "TiedLMHead",
                                self.logits(c, t), 1)
            for t in range(p.tp):
                yield self._rec(dr, c, t, mb, "ActivationGradIn", "model.lm_head", "TiedLMHead",
                                self.hidden(c, t, p.sp), rep if p.sp else p.tp)
        for c, t in self.ranks:
            for kind in ("ActivationGradOut", "ActivationGradIn"):
                yield self._rec(dr, c, t, mb, kind, "model.final_norm", "LayerNorm",
                                self.hidden(c, t, True), rep)
        for layer in reversed(range(m.layers)):
            for name, cls in ((f"model.layers.{layer}.mlp", "MlpBlock"),
                              (f"model.layers.{layer}.attn", "AttentionBlock")):
                for c in range(p.cp):
                    for t in range(p.tp):
                        yield self._rec(dr, c, t, mb, "ActivationGradOut", name, cls,
                                        self.hidden(c, t, True), rep)
                for c in range(p.cp):
                    for t in range(p.tp):
                        yield self._rec(dr, c, t, mb, "ActivationGradIn", name, cls,
                                        self.hidden(c, t, True), rep)
        for c in range(p.cp):
            for t in range(p.tp):
                yield self._rec(dr, c, t, mb, "ActivationGradOut", "model.embedding", "Embedding",
                                self.hidden(c, t, True), rep)
        if p.cp > 1:
            return  # per-microbatch grads under cp have no shard interpretation (engine.py:928-931)
        for path, shape in self.params:
            if p.sp and is_norm_param(path):
                continue
            for c, t in self.ranks:
                if path.endswith(".position"):
                    mapping, replica = self.position_grad(c, t), (1 if p.sp else p.tp)
                else:
                    mapping = self.param(path, shape, t)
                    replica = p.tp if param_tp_axis(path) is None else 1
                yield self._rec(dr, c, t, mb, "ParamGrad", path, "Param", mapping, replica)

    def _main_grads(self):
        p = self.p
        for path, shape in self.params:
            sharded = param_tp_axis(path) is not None
            replica = p.dp * p.cp * (1 if sharded else p.tp)
            for dr in range(p.dp):
                for c in range(p.cp):
                    for t in range(p.tp):
                        yield self._rec(dr, c, t, 0, "MainGrad", path, "Param",
                                        self.param(path, shape, t), replica)

    def records(self):
        """Every record of one training iteration, in execution order
        (engine.py:966-979)."""
        p = self.p
        yield from self._params(self.iteration)
        per_dp = p.microbatches // p.dp
        for dr in range(p.dp):
            for local in range(per_dp):
                mb = dr * per_dp + local
                yield from self._forward(dr, mb)
                yield from self._backward(dr, mb)
        yield from self._main_grads()
        yield from self._params(self.iteration + 1)


def emit_records(m: ModelShape, p: ParallelConfig, iteration: int = 0) -> list[RecordSpec]:
    return list(Layout(m, p, iteration).records())


# named model shapes of the benchmark configs (BASELINE.json configs)
GPT2_SMALL_L2 = ModelShape(layers=2, d_model=768, n_heads=12, d_ff=3072, seq_len=1024, vocab=50304)
GPT2_MEDIUM = ModelShape(layers=24, d_model=1024, n_heads=16, d_ff=4096, seq_len=1024, vocab=50304)
LLAMA3_1B = ModelShape(layers=16, d_model=2048, n_heads=32, d_ff=8192, seq_len=8192, vocab=128256,
                       n_kv_heads=8, gated_mlp=True, norm_bias=False, position_table=False)
LLAMA3_8B = ModelShape(layers=32, d_model=4096, n_heads=32, d_ff=14336, seq_len=8192, vocab=128256,
                       n_kv_heads=8, gated_mlp=True, norm_bias=False, position_table=False)


# -- execution order of a trace split across ranks ------------------------------

_PARAM_SLOTS = {"attn.norm.weight": 0, "attn.norm.bias": 1, "attn.wq": 2, "attn.wk": 3, "attn.wv": 4,
                "attn.wo": 5, "mlp.norm.weight": 6, "mlp.norm.bias": 7, "mlp.w1": 8, "mlp.w3": 9,
                "mlp.w2": 10}
_BIG = 1 << 40


def _module_index(module: str):
    """Forward position of a traced module: embedding, then per layer attn
    and mlp, then final_norm and lm_head (engine.py:971-975)."""
    if module == "model.embedding":
        return 0
    if module == "model.final_norm":
        return _BIG
    if module == "model.lm_head":
        return _BIG + 1
    parts = module.split(".")
    if len(parts) == 4 and parts[0] == "model" and parts[1] == "layers" and parts[2].isdigit() \
            and parts[3] in ("attn", "mlp"):
        return 1 + 2 * int(parts[2]) + (parts[3] == "mlp")
    return None


def _param_index(path: str):
    """Registration position of a parameter path (param_shapes order)."""
    if path == "model.embedding.word":
        return (0, 0, 0)
    if path == "model.embedding.position":
        return (0, 0, 1)
    if path == "model.final_norm.weight":
        return (2, 0, 0)
    if path == "model.final_norm.bias":
        return (2, 0, 1)
    parts = path.split(".", 3)
    if len(parts) == 4 and parts[0] == "model" and parts[1] == "layers" and parts[2].isdigit():
        slot = _PARAM_SLOTS.get(parts[3])
        if slot is not None:
            return (1, int(parts[2]), slot)
    return None


_FWD = {"ActivationIn": 0, "ActivationOut": 1}
_BWD = {"ActivationGradOut": 0, "ActivationGradIn": 1}


def execution_key(ident, rank_meta):
    """Sort key that puts the records of a trace split across ranks (PP
    stages, CP/DP/TP ranks) back into the single-process execution order of
    the reference schedule (Emulator.run_iteration, engine.py:966-979; the
    order Layout.records emits): Param of the iteration, then per microbatch
    its forward (modules in order, ActivationIn before ActivationOut), its
    backward (modules reversed, GradOut before GradIn) and its ParamGrads
    (registration order), then MainGrad, then the next iteration's Param;
    copies of one id in (dp, cp, tp) rank order.  The order of first
    occurrences is the report order (checker.py:205-206) and the order
    within an id picks each replica group's copy 0 (checker.py:184-191).
    None when the id is not one of the reference model's modules or
    parameters (then the caller keeps rank-major order)."""
    kind, module = ident.kind.value, ident.module_name
    rank = (rank_meta.dp, rank_meta.cp, rank_meta.tp)
    if kind in ("Param", "MainGrad"):
        p = _param_index(module)
        if p is None:
            return None
        return (ident.iteration, 0 if kind == "Param" else 2, 0, 0, p, rank)
    if kind == "ParamGrad":
        p = _param_index(module)
        return None if p is None else (ident.iteration, 1, ident.microbatch, 2, p, rank)
    m = _module_index(module)
    if m is None:
        return None
    if kind in _FWD:
        return (ident.iteration, 1, ident.microbatch, 0, (m, _FWD[kind]), rank)
    if kind in _BWD:
        return (ident.iteration, 1, ident.microbatch, 1, (-m, _BWD[kind]), rank)
    return None
