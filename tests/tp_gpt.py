"""A live Megatron-style tensor-parallel GPT in plain PyTorch — TEST
INFRASTRUCTURE for §8(f) #3 (real-TP annotated captures).

The architecture is the reference model's (pkg/src/traindiff/model.py:
token + learned position embedding, `layers` x (Pre-LN attention block,
Pre-LN MLP block) with residual adds and bias-free projections, final
LayerNorm, weight-tied LM head, mean next-token cross-entropy with labels
rolled left by one), with the module names the reference traces
(`model.embedding`, `model.layers.{i}.attn|mlp`, `model.final_norm`,
`model.lm_head`) and its parameter layout (y = x @ W, W stored (in, out)).

Tensor parallelism follows the reference emulator's TP geometry
(engine.py:210-222, 420-529): vocab-parallel `word` (axis 0) with an
all-reduce of the lookup partials, column-parallel `wq/wk/wv/w1` (axis 1),
row-parallel `wo/w2` (axis 0) followed by an all-reduce, replicated norms
and position table; the LM head produces vocab-parallel logits and the loss
is a vocab-parallel cross-entropy.  The collectives are real
torch.distributed calls (gloo here, on host or CUDA tensors), wrapped as the
usual Megatron `f` / `g` autograd pair so the backward all-reduces the
column-parallel input gradients.

`skip_reduce` names blocks whose row-parallel all-reduce is dropped — the
reference's MC_TP_ROW_ALLREDUCE injection (engine.py:504-529): each rank
then keeps its partial sum and the block output's replicas disagree.

shape["llama"] = True switches to the Llama-3 block the B200 layout rules
extend the reference to (layout.py: `gated_mlp`, `n_kv_heads`,
`norm_bias=False`, `position_table=False`): RMSNorm without bias, GQA with
shape["kv_heads"] key/value heads (column-parallel by KV head), rotary
position (no table), SwiGLU MLP with a column-parallel `w3`.  A live run of
it pins those emission rules: every capture must fit the shard map
layout_shard assigns it, and the TP run must agree with one device.
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


class TPGroup:
    """The TP communicator of one rank (world 1 = single device, no calls)."""

    def __init__(self, rank: int = 0, world: int = 1, group=None):
        self.rank, self.world, self.group = rank, world, group

    def all_reduce_(self, t: torch.Tensor, op: str = "sum") -> torch.Tensor:
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX,
                            group=self.group)
        return t


class _CopyToTP(torch.autograd.Function):
    """Megatron `f`: identity forward, all-reduce of the gradient backward."""

    @staticmethod
    def forward(ctx, x, g):
        ctx.g = g
        return x.clone()

    @staticmethod
    def backward(ctx, dy):
        return ctx.g.all_reduce_(dy.contiguous().clone()), None


class _ReduceFromTP(torch.autograd.Function):
    """Megatron `g`: all-reduce forward, identity backward."""

    @staticmethod
    def forward(ctx, x, g):
        return g.all_reduce_(x.contiguous().clone())

    @staticmethod
    def backward(ctx, dy):
        return dy, None


def full_params(shape: dict, seed: int = 1234, std: float = 0.02) -> dict:
    """Deterministic full (unsharded) fp32 parameters, registration order of
    model.param_specs (depth-scaled std on the residual output projections)."""
    gen = torch.Generator().manual_seed(seed)
    d, ff, L, V, S = shape["d"], shape["ff"], shape["layers"], shape["vocab"], shape["seq"]
    llama = shape.get("llama", False)
    kv = d // shape["heads"] * shape.get("kv_heads", shape["heads"])
    res_std = std / math.sqrt(2.0 * L)
    out = {"model.embedding.word": torch.randn(V, d, generator=gen) * std}
    if not llama:
        out["model.embedding.position"] = torch.randn(S, d, generator=gen) * std
    for i in range(L):
        a, m = f"model.layers.{i}.attn", f"model.layers.{i}.mlp"
        out[f"{a}.wq"] = torch.randn(d, d, generator=gen) * std
        for w in ("wk", "wv"):
            out[f"{a}.{w}"] = torch.randn(d, kv, generator=gen) * std
        out[f"{a}.wo"] = torch.randn(d, d, generator=gen) * res_std
        out[f"{m}.w1"] = torch.randn(d, ff, generator=gen) * std
        if llama:
            out[f"{m}.w3"] = torch.randn(d, ff, generator=gen) * std
        out[f"{m}.w2"] = torch.randn(ff, d, generator=gen) * res_std
    return out


def _norm(d: int, llama: bool):
    return torch.nn.RMSNorm(d, eps=1e-5) if llama else torch.nn.LayerNorm(d, eps=1e-5)


def _rotary(x):
    """Rotary position embedding of (heads, S, dh), half-split pairs."""
    h, S, dh = x.shape
    half = dh // 2
    inv = 1.0 / (10000.0 ** (torch.arange(half, device=x.device, dtype=torch.float32) / half))
    ang = torch.arange(S, device=x.device, dtype=torch.float32)[:, None] * inv[None, :]
    cos, sin = ang.cos().to(x.dtype), ang.sin().to(x.dtype)
    a, b = x[..., :half], x[..., half:]
    return torch.cat([a * cos - b * sin, a * sin + b * cos], dim=-1)


def _shard(w: torch.Tensor, axis: int, g: TPGroup) -> torch.Tensor:
    n = w.shape[axis] // g.world
    return w.narrow(axis, g.rank * n, n).clone()


class Embedding(torch.nn.Module):
    def __init__(self, word, position, g: TPGroup):
        super().__init__()
        self.g = g
        self.word = torch.nn.Parameter(_shard(word, 0, g))
        if position is not None:
            self.position = torch.nn.Parameter(position.clone())
        else:
            self.position = None

    def forward(self, ids):
        v = self.word.shape[0]
        local = ids - self.g.rank * v
        inside = (local >= 0) & (local < v)
        rows = F.embedding(local.clamp(0, v - 1), self.word) * inside[:, None].to(self.word.dtype)
        out = _ReduceFromTP.apply(rows, self.g)
        return out + self.position if self.position is not None else out


class AttentionBlock(torch.nn.Module):
    def __init__(self, name, P, n_heads, g: TPGroup, skip_reduce=False, llama=False):
        super().__init__()
        d = P[f"{name}.wq"].shape[0]
        self.g, self.skip_reduce, self.llama = g, skip_reduce, llama
        self.heads, self.dh = n_heads // g.world, d // n_heads
        self.kv_heads = P[f"{name}.wk"].shape[1] // self.dh // g.world
        self.norm = _norm(d, llama)
        for w in ("wq", "wk", "wv"):
            setattr(self, w, torch.nn.Parameter(_shard(P[f"{name}.{w}"], 1, g)))
        self.wo = torch.nn.Parameter(_shard(P[f"{name}.wo"], 0, g))

    def forward(self, x):
        S = x.shape[0]
        a = _CopyToTP.apply(self.norm(x), self.g)
        q = (a @ self.wq).view(S, self.heads, self.dh).transpose(0, 1)
        k, v = ((a @ w).view(S, self.kv_heads, self.dh).transpose(0, 1) for w in (self.wk, self.wv))
        if self.llama:
            q, k = _rotary(q), _rotary(k)
        if self.kv_heads != self.heads:         # GQA: each KV head serves heads/kv_heads queries
            k = k.repeat_interleave(self.heads // self.kv_heads, dim=0)
            v = v.repeat_interleave(self.heads // self.kv_heads, dim=0)
        o = F.scaled_dot_product_attention(q[None], k[None], v[None], is_causal=True)[0]
        y = o.transpose(0, 1).reshape(S, self.heads * self.dh) @ self.wo
        if not self.skip_reduce:
            y = _ReduceFromTP.apply(y, self.g)
        return x + y


class MlpBlock(torch.nn.Module):
    def __init__(self, name, P, g: TPGroup, skip_reduce=False, llama=False):
        super().__init__()
        d = P[f"{name}.w1"].shape[0]
        self.g, self.skip_reduce, self.llama = g, skip_reduce, llama
        self.norm = _norm(d, llama)
        self.w1 = torch.nn.Parameter(_shard(P[f"{name}.w1"], 1, g))
        if llama:
            self.w3 = torch.nn.Parameter(_shard(P[f"{name}.w3"], 1, g))
        self.w2 = torch.nn.Parameter(_shard(P[f"{name}.w2"], 0, g))

    def forward(self, x):
        a = _CopyToTP.apply(self.norm(x), self.g)
        if self.llama:
            y = (F.silu(a @ self.w1) * (a @ self.w3)) @ self.w2
        else:
            y = F.gelu(a @ self.w1, approximate="tanh") @ self.w2
        if not self.skip_reduce:
            y = _ReduceFromTP.apply(y, self.g)
        return x + y


class Layer(torch.nn.Module):
    def __init__(self, i, P, n_heads, g, skip, llama=False):
        super().__init__()
        self.attn = AttentionBlock(f"model.layers.{i}.attn", P, n_heads, g, f"model.layers.{i}.attn" in skip,
                                   llama)
        self.mlp = MlpBlock(f"model.layers.{i}.mlp", P, g, f"model.layers.{i}.mlp" in skip, llama)

    def forward(self, x):
        return self.mlp(self.attn(x))


class TiedLMHead(torch.nn.Module):
    """Vocab-parallel logits against the (tied) word-embedding shard."""

    def __init__(self, embedding: Embedding, g: TPGroup):
        super().__init__()
        self._emb = [embedding]          # not a sub-module: the weight is embedding.word
        self.g = g

    def forward(self, h):
        return _CopyToTP.apply(h, self.g) @ self._emb[0].word.t()


class TPGPT(torch.nn.Module):
    def __init__(self, shape: dict, g: TPGroup, params: dict | None = None, skip_reduce=()):
        super().__init__()
        P = params if params is not None else full_params(shape)
        llama = shape.get("llama", False)
        self.g = g
        self.embedding = Embedding(P["model.embedding.word"], P.get("model.embedding.position"), g)
        self.layers = torch.nn.ModuleList(Layer(i, P, shape["heads"], g, set(skip_reduce), llama)
                                          for i in range(shape["layers"]))
        self.final_norm = _norm(shape["d"], llama)
        self.lm_head = TiedLMHead(self.embedding, g)

    def forward(self, ids):
        h = self.embedding(ids)
        for layer in self.layers:
            h = layer(h)
        return self.lm_head(self.final_norm(h))

    def loss(self, ids):
        """Mean next-token cross-entropy over vocab-parallel logits."""
        logits = self(ids).float()
        labels = torch.roll(ids, -1)
        v = logits.shape[1]
        with torch.no_grad():
            m = self.g.all_reduce_(logits.max(dim=1).values.clone(), "max")
        sumexp = _ReduceFromTP.apply((logits - m[:, None]).exp().sum(dim=1), self.g)
        local = labels - self.g.rank * v
        inside = (local >= 0) & (local < v)
        tgt = logits.gather(1, local.clamp(0, v - 1)[:, None])[:, 0] * inside.to(logits.dtype)
        tgt = _ReduceFromTP.apply(tgt, self.g)
        return (sumexp.log() + m - tgt).mean()


# tap patterns: the reference's traced modules plus the block norms (for
# their ParamGrads; their activations get the block's hidden map)
PATTERNS = ("embedding", "layers.*.attn", "layers.*.attn.norm", "layers.*.mlp",
            "layers.*.mlp.norm", "final_norm", "lm_head")


def model_shape(shape: dict):
    from paper_2506_09280_b200.layout import ModelShape
    llama = shape.get("llama", False)
    return ModelShape(layers=shape["layers"], d_model=shape["d"], n_heads=shape["heads"],
                      d_ff=shape["ff"], seq_len=shape["seq"], vocab=shape["vocab"],
                      n_kv_heads=shape.get("kv_heads"), gated_mlp=llama, norm_bias=not llama,
                      position_table=not llama)


def traced_step(shape: dict, g: TPGroup, *, device="cpu", dtype=torch.float32, skip_reduce=(),
                perturb=None, precision="fp32", seed_tokens: int = 99, dp: int = 1, dp_rank: int = 0,
                microbatch: int = 0):
    """One forward+backward of TP rank g.rank (of DP rank dp_rank when the
    job is dp x tp), traced with that rank's real maps
    (torchtap.layout_shard) under microbatch `microbatch` (its tokens are
    seeded by seed_tokens + microbatch).  perturb(tensor, ident) -> tensor
    is applied to the embedding output (the reference's perturbation site,
    engine.py:466-471).  Returns the TapHandle."""
    from paper_2506_09280_b200 import torchtap
    from paper_2506_09280_b200.layout import Layout, ParallelConfig
    model = TPGPT(shape, g, skip_reduce=skip_reduce).to(device=device, dtype=dtype)
    layout = Layout(model_shape(shape), ParallelConfig(tp=g.world, dp=dp, microbatches=dp))
    cfg = torchtap.TapConfig(patterns=PATTERNS, precision=precision, microbatch=microbatch,
                             shard=torchtap.layout_shard(layout, dp=dp_rank, tp=g.rank))
    handle = torchtap.attach(model, cfg)
    if perturb is not None:
        ident = f"iter=0|mb={microbatch}|kind=ActivationOut|mod=model.embedding"
        # prepended: runs before the tap's output hook, which then captures
        # (and the model consumes) the perturbed embedding output
        from paper_2506_09280_b200.perturb import straight_through
        model.embedding.register_forward_hook(lambda mod, args, out: straight_through(out, perturb(out, ident)),
                                              prepend=True)
    ids = torch.randint(0, shape["vocab"], (shape["seq"],),
                        generator=torch.Generator().manual_seed(seed_tokens + microbatch)).to(device)
    model.loss(ids).backward()
    torchtap.detach(handle)
    return handle
