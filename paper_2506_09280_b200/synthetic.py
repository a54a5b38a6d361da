"""Synthetic traces of the named model shapes, built directly in HBM.

The reference is the single-device layout (identity mappings) of `model`;
the candidate is `pcfg`'s layout from layout.emit_records.  Values: the
reference tensor of each id is N(0, sigma_kind) rounded to the storage
dtype; the candidate's logical tensor is Q(ref * (1 + eps*u)) with u from
the counter-based stream tagged "cand|{id}" (td_perturb — simulated
round-off), and each candidate record holds its shard of it, laid out
through its own ShardMapping (replicas are separate allocations, so every
copy is real memory traffic).  Optional bugs corrupt chosen ids the way the
config-3 injections do (wrong shard order, missing allreduce, scale error).
"""

from __future__ import annotations

from .canonical import identity_mapping, parse_canonical
from .layout import ModelShape, ParallelConfig, emit_records
from .perturb import PerturbSpec, apply_perturbation
from .tracestore import RankMeta, Trace, TraceRecord

SIGMA = {"Param": 0.02, "MainGrad": 1e-3, "ParamGrad": 1e-3, "ActivationGradIn": 1e-3,
         "ActivationGradOut": 1e-3}


def _sigma(kind: str) -> float:
    return SIGMA.get(kind, 1.0)


def _fill(shape, kind, vocab, gen, dtype):
    import torch
    if kind == "ActivationIn" and len(shape) == 1:
        # token ids entering the embedding
        return torch.randint(0, vocab, shape, generator=gen, device="cuda").to(dtype)
    return (torch.randn(shape, generator=gen, device="cuda") * _sigma(kind)).to(dtype)


def _shard(full, mapping):
    import torch
    out = torch.empty(mapping.local_shape, dtype=full.dtype, device=full.device)
    for loc, glob in mapping.pairs:
        out[loc.as_slices()] = full[glob.as_slices()]
    return out


def build(model: ModelShape, pcfg: ParallelConfig, *, dtype=None, seed: int = 0,
          eps: float = 2.0 ** -8, bugs: dict | None = None, header: dict | None = None):
    """(reference trace, candidate trace), payloads resident in HBM.

    bugs: {id_string: "scale" | "order" | "partial"} corruptions of the
    candidate (scale error x tp; TP shards swapped under unchanged maps;
    per-rank partial sums left unreduced)."""
    import torch
    dtype = dtype or torch.bfloat16
    bugs = bugs or {}
    hdr = header or {"digest": f"synthetic-{model}-{seed}", "mode": "cascade"}
    ref_specs = emit_records(model, ParallelConfig(microbatches=pcfg.microbatches))
    cand_specs = emit_records(model, pcfg)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    ref = Trace(header=dict(hdr))
    full: dict = {}
    policy = "bf16" if dtype == torch.bfloat16 else "fp32"
    for s in ref_specs:
        kind = s.ident.split("|")[2][5:]
        x = _fill(s.mapping.global_shape, kind, model.vocab, gen, dtype)
        ref.records.append(TraceRecord(parse_canonical(s.ident), RankMeta(*s.rank), s.mapping,
                                       s.replica, x, s.module_class))
        full[s.ident] = x
    cand = Trace(header=dict(hdr))
    cand_full: dict = {}
    order: dict = {}
    for s in cand_specs:
        if s.ident not in cand_full:
            x = full.get(s.ident)
            if x is None:
                kind = s.ident.split("|")[2][5:]
                x = _fill(s.mapping.global_shape, kind, model.vocab, gen, dtype)
            shape = x.shape
            y = x if x.dim() == 0 else apply_perturbation(
                x.reshape(-1, shape[-1]) if x.dim() > 1 else x.reshape(1, -1),
                "cand|" + s.ident, PerturbSpec(0, eps), policy=policy).reshape(shape)
            if bugs.get(s.ident) == "scale":
                y = (y.float() * pcfg.tp).to(dtype)
            cand_full[s.ident] = y
        y = cand_full[s.ident]
        payload = _shard(y, s.mapping)
        bug = bugs.get(s.ident)
        if bug == "order":
            order.setdefault(s.ident, []).append(len(cand.records))
        if bug == "partial" and payload.numel():
            payload = (payload.float() / pcfg.tp * (1 + s.rank[1])).to(dtype)
        cand.records.append(TraceRecord(parse_canonical(s.ident), RankMeta(*s.rank), s.mapping,
                                        s.replica, payload, s.module_class))
    for ident, idx in order.items():
        # swap the first two TP shards' payloads under unchanged maps
        if len(idx) >= 2:
            a, b = cand.records[idx[0]], cand.records[idx[1]]
            if a.shape == b.shape:
                a.payload, b.payload = b.payload, a.payload
    return ref, cand


def flat_tolerances(trace, value: float) -> dict:
    return {rec.id.encode(): value for rec in trace.records}


def sweep_pair(n_bytes: int, *, maps: str = "identity", g: int = 1, dtype=None, seed: int = 0,
               eps: float = 2.0 ** -8):
    """Config 5: one id of n_bytes per tensor, shape (N/4096, 4096), candidate
    split `g` ways by columns ("columns") or CP-striped in 2 pairs ("stripes")."""
    import torch
    from .canonical import CanonicalId, ShardMapping, SliceBox, TensorKind
    dtype = dtype or torch.bfloat16
    esize = torch.tensor([], dtype=dtype).element_size()
    cols = 4096
    rows = max(1, n_bytes // esize // cols)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((rows, cols), generator=gen, device="cuda").to(dtype)
    ident = CanonicalId(0, 0, TensorKind.ACTIVATION_OUT, f"sweep.{n_bytes}")
    hdr = {"digest": "sweep", "mode": "cascade"}
    ref = Trace(hdr, [TraceRecord(ident, RankMeta(), identity_mapping((rows, cols)), 1, x, "Sweep")])
    y = apply_perturbation(x, "cand|" + ident.encode(), PerturbSpec(0, eps),
                           policy="bf16" if dtype == torch.bfloat16 else "fp32")
    cand = Trace(hdr, [])
    if maps == "identity":
        cand.records.append(TraceRecord(ident, RankMeta(), identity_mapping((rows, cols)), 1, y, "Sweep"))
    elif maps == "columns":
        w = cols // g
        for t in range(g):
            m = ShardMapping((rows, w), (rows, cols),
                             ((SliceBox(((0, rows), (0, w))), SliceBox(((0, rows), (t * w, (t + 1) * w)))),))
            cand.records.append(TraceRecord(ident, RankMeta(tp=t), m, 1, _shard(y, m), "Sweep"))
    elif maps == "stripes":
        ch = rows // (2 * g)
        for c in range(g):
            pieces = [((0, ch), (c * ch, (c + 1) * ch)),
                      ((ch, 2 * ch), ((2 * g - 1 - c) * ch, (2 * g - c) * ch))]
            pairs = tuple((SliceBox((l, (0, cols))), SliceBox((gg, (0, cols)))) for l, gg in pieces)
            m = ShardMapping((2 * ch, cols), (rows, cols), pairs)
            cand.records.append(TraceRecord(ident, RankMeta(cp=c), m, 1, _shard(y, m), "Sweep"))
    else:
        raise ValueError(maps)
    return ref, cand


class ShareLayout:
    """Every GPU's share of a multi-GPU job, as metadata (no payloads).

    Candidate record r lives on owner(r) (default: (dp, tp) -> dp*tp_size +
    tp, cp ranks after, mod world).  The compare of each candidate shard group
    runs where the copy plan.compare_copies picks lives (copy 0, or the
    least-loaded holder of a cross-rank replica group), and that rank also
    holds the reference slices covering the group's global boxes — what
    distributed.split_reference hands it.  `records(rank)` is the ordered
    content of one rank's (reference, candidate) traces, `metas()` the
    RecordMeta lists every rank would publish, so one process can build the
    global plan of a job whose other ranks are not present (bench config 4)."""

    def __init__(self, model: ModelShape, pcfg: ParallelConfig, world: int, owner=None,
                 dtype_code: int = 1):
        from .canonical import ShardMapping, SliceBox
        from .distributed import RecordMeta, _MetaTrace, sort_metas
        from .layout import execution_key
        from .plan import compare_copies, merge_view
        self.model, self.pcfg, self.world = model, pcfg, world
        self.owner = owner or (lambda s: (s.rank[0] * pcfg.tp + s.rank[1] + pcfg.tp * pcfg.dp * s.rank[4]) % world)
        self.ref_specs = {s.ident: s for s in emit_records(model, ParallelConfig(microbatches=pcfg.microbatches))}
        self.cand_specs = emit_records(model, pcfg)
        self.ids: dict = {}                      # ident -> generation index
        for spec in self.cand_specs:
            self.ids.setdefault(spec.ident, len(self.ids))
        # candidate: each rank's records in emission order
        self.cand = [[] for _ in range(world)]   # [(ident, spec)]
        metas = []
        for spec in self.cand_specs:
            o = self.owner(spec)
            pos = len(self.cand[o])
            self.cand[o].append((spec.ident, spec))
            ident, rank = parse_canonical(spec.ident), RankMeta(*spec.rank)
            metas.append(RecordMeta(ident, rank, spec.mapping, spec.replica, tuple(spec.mapping.local_shape),
                                    dtype_code, spec.module_class, o, (o, pos), None,
                                    execution_key(ident, rank)))
        sort_metas(metas)            # the order global_trace() gives the live job
        view = merge_view(_MetaTrace({}, metas))
        choice = compare_copies(view, lambda m: m.owner)
        # reference slices: for every compared group, its global boxes on the
        # compare holder, numbered per id across all ranks (distinct rank
        # metadata per piece, as split_reference does)
        self.ref = [[] for _ in range(world)]    # [(ident, piece k, ShardMapping, module class)]
        for ident, meta in view.items():
            rspec = self.ref_specs.get(ident)
            if rspec is None or not meta.merge_ok or meta.global_shape != rspec.mapping.global_shape:
                continue
            shape = rspec.mapping.global_shape
            k = 0
            for gi, g in enumerate(meta.groups):
                holder = g.records[choice.get((ident, gi), 0)]
                for _, gbox in holder.mapping.pairs:
                    ext = gbox.extents
                    local = SliceBox(tuple((0, e) for e in ext))
                    self.ref[holder.owner].append(
                        (ident, k, ShardMapping(ext, shape, ((local, gbox),)), rspec.module_class))
                    k += 1

    def metas(self, dtype_code: int = 1) -> tuple[list, list]:
        """(reference metas per rank, candidate metas per rank): what each
        rank's global_trace() publishes, in its local record order."""
        from .distributed import RecordMeta
        from .layout import execution_key

        def meta(i, rank, m, rep, mc, r, pos):
            ident = parse_canonical(i)
            return RecordMeta(ident, rank, m, rep, tuple(m.local_shape), dtype_code, mc, r, (r, pos), None,
                              execution_key(ident, rank))
        ref = [[meta(i, RankMeta(0, k, 0, 0, 0, 0), m, 1, mc, r, pos) for pos, (i, k, m, mc) in enumerate(self.ref[r])]
               for r in range(self.world)]
        cand = [[meta(i, RankMeta(*s.rank), s.mapping, s.replica, s.module_class, r, pos)
                 for pos, (i, s) in enumerate(self.cand[r])] for r in range(self.world)]
        return ref, cand

    def build(self, rank: int, *, dtype=None, seed: int = 0, eps: float = 2.0 ** -8,
              header: dict | None = None, bugs: dict | None = None):
        """(reference trace, candidate trace) of `rank`, payloads in HBM.
        Values: as build() — every rank draws an id's logical tensors from
        the same seed, so shards on different ranks fit together.  bugs: as
        build()'s ("scale" / "order" / "partial"), applied to the records
        wherever they live ("order" swaps the id's first two TP shards'
        payloads across ranks: each holder cuts its record through the
        partner's map)."""
        import torch
        dtype = dtype or torch.bfloat16
        bugs = bugs or {}
        hdr = header or {"digest": f"synthetic-{self.model}-{seed}", "mode": "cascade"}
        policy = "bf16" if dtype == torch.bfloat16 else "fp32"
        partner: dict = {}                  # id(spec) -> spec whose map cuts its payload
        for ident, bug in bugs.items():
            if bug != "order":
                continue
            specs = [sp for sp in self.cand_specs if sp.ident == ident][:2]
            if len(specs) == 2 and tuple(specs[0].mapping.local_shape) == tuple(specs[1].mapping.local_shape):
                partner[id(specs[0])], partner[id(specs[1])] = specs[1], specs[0]
        ref, cand = Trace(header=dict(hdr)), Trace(header=dict(hdr))
        need = {i for i, _ in self.cand[rank]} | {i for i, *_ in self.ref[rank]}
        cand_by_id: dict = {}
        for pos, (ident, spec) in enumerate(self.cand[rank]):
            cand_by_id.setdefault(ident, []).append(pos)
        ref_by_id: dict = {}
        for pos, entry in enumerate(self.ref[rank]):
            ref_by_id.setdefault(entry[0], []).append(pos)
        cand_recs = [None] * len(self.cand[rank])
        ref_recs = [None] * len(self.ref[rank])
        gen = torch.Generator(device="cuda")
        for ident in sorted(need, key=self.ids.__getitem__):
            gen.manual_seed(seed * 1000003 + self.ids[ident])
            rspec = self.ref_specs.get(ident)
            shape = rspec.mapping.global_shape if rspec else \
                self.cand[rank][cand_by_id[ident][0]][1].mapping.global_shape
            kind = ident.split("|")[2][5:]
            x = _fill(shape, kind, self.model.vocab, gen, dtype)
            if ident in cand_by_id:
                y = x if x.dim() == 0 else apply_perturbation(
                    x.reshape(-1, shape[-1]) if x.dim() > 1 else x.reshape(1, -1),
                    "cand|" + ident, PerturbSpec(0, eps), policy=policy).reshape(shape)
                if bugs.get(ident) == "scale":
                    y = (y.float() * self.pcfg.tp).to(dtype)
                for pos in cand_by_id[ident]:
                    s = self.cand[rank][pos][1]
                    payload = _shard(y, partner.get(id(s), s).mapping)
                    if bugs.get(ident) == "partial" and payload.numel():
                        payload = (payload.float() / self.pcfg.tp * (1 + s.rank[1])).to(dtype)
                    cand_recs[pos] = TraceRecord(parse_canonical(ident), RankMeta(*s.rank), s.mapping,
                                                 s.replica, payload, s.module_class)
                del y
            for pos in ref_by_id.get(ident, ()):
                _, k, m, mc = self.ref[rank][pos]
                gbox = m.pairs[0][1]
                ref_recs[pos] = TraceRecord(parse_canonical(ident), RankMeta(0, k, 0, 0, 0, 0), m, 1,
                                            x[gbox.as_slices()].contiguous(), mc)
            del x
        ref.records, cand.records = ref_recs, cand_recs
        return ref, cand


def build_rank_share(model: ModelShape, pcfg: ParallelConfig, world: int, rank: int, *,
                     owner=None, dtype=None, seed: int = 0, eps: float = 2.0 ** -8,
                     header: dict | None = None):
    """One GPU's share of a multi-GPU job, built without materialising the
    others' (see ShareLayout).  Returns (ref_local, cand_local, layout)."""
    layout = ShareLayout(model, pcfg, world, owner)
    ref, cand = layout.build(rank, dtype=dtype, seed=seed, eps=eps, header=header)
    return ref, cand, layout
