"""Multi-GPU check: one process per GPU, partial sums across NVLink.

SURVEY §8(e).  A canonical id's compare is a sum over disjoint boxes, so:

1. every rank publishes the METADATA of the records it holds (ids, maps,
   replica sizes, dtypes, shapes — no payload) with one all_gather_object;
   all ranks then hold the same global merge view (host, deterministic);
2. each rank plans only the work whose operands it holds (plan.Plan with
   owner/me): compare runs on the rank holding the candidate's copy 0 (its
   reference slice must be local), replica sums fused when a group's copies
   are all on that rank;
3. replica groups whose copies live on several ranks are decided by 128-bit
   order-independent digests (td_fingerprint: every local copy in one
   launch; one int64 all_reduce of a small table): equal digests = identical
   copies = rel_err 0, so the group's slot stays zero, and the group's
   compare may read any copy — plan.compare_copies spreads those compares
   over the holders to balance bytes per GPU; on a mismatch (the bug path
   only) the differing copies are sent point-to-point to copy 0's rank,
   which computes the exact rel_err sums, and a compare that read another
   copy is handed copy 0 instead;
4. ONE all_reduce(sum, f64) of the per-id / per-group slot vector crosses
   NVLink, then every rank runs td_verdict on identical sums and can render
   the report.

`Comm` abstracts the collectives: `TorchComm` wraps torch.distributed (NCCL
on the GPU box, gloo for the CPU tests); `ThreadComm` runs N logical ranks
as threads of one process on one GPU, so the whole algorithm — kernels
included — is testable where only one GPU exists.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N


# ---------------------------------------------------------------------------
# communicators

class Comm:
    rank: int
    world: int

    def all_gather_object(self, obj) -> list:
        raise NotImplementedError

    def all_reduce_sum_(self, tensor) -> None:
        raise NotImplementedError

    def exchange(self, sends: list, recvs: list) -> None:
        """sends: [(dst, tensor)], recvs: [(src, tensor)] — matched in order."""
        raise NotImplementedError


class TorchComm(Comm):
    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather_object(self, obj) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def all_reduce_sum_(self, tensor) -> None:
        self.dist.all_reduce(tensor, op=self.dist.ReduceOp.SUM, group=self.group)

    def exchange(self, sends, recvs) -> None:
        ops = [self.dist.P2POp(self.dist.isend, t, self._g(d), self.group) for d, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t, self._g(s), self.group) for s, t in recvs]
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def _g(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)


class _ThreadHub:
    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.mail: dict = {}


class ThreadComm(Comm):
    """N logical ranks as threads of one process (tests on a single GPU)."""

    def __init__(self, hub: _ThreadHub, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    @staticmethod
    def hub(world: int) -> _ThreadHub:
        return _ThreadHub(world)

    def _sync(self):
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        self.hub.barrier.wait()

    def all_gather_object(self, obj) -> list:
        self.hub.slots[self.rank] = obj
        self._sync()
        out = list(self.hub.slots)
        self._sync()
        return out

    def all_reduce_sum_(self, tensor) -> None:
        self.hub.slots[self.rank] = tensor.clone()
        self._sync()
        total = self.hub.slots[0].clone()
        for t in self.hub.slots[1:]:
            total += t
        tensor.copy_(total)
        self._sync()

    def exchange(self, sends, recvs) -> None:
        for k, (dst, t) in enumerate(sends):
            self.hub.mail[(self.rank, dst, k)] = t
        self._sync()
        counters: dict = {}
        for src, t in recvs:
            k = counters.get(src, 0)
            # sends from `src` to me are numbered in src's send order, skipping other dsts
            mine = sorted(key for key in self.hub.mail if key[0] == src and key[1] == self.rank)
            t.copy_(self.hub.mail[mine[k]])
            counters[src] = k + 1
        self._sync()
        if self.rank == 0:
            self.hub.mail.clear()
        self._sync()


class StaticComm(Comm):
    """A rank of a job whose record metadata is known in advance
    (synthetic.ShareLayout): all_gather_object answers from the precomputed
    per-rank lists (one list of lists per call, in call order), reductions
    and exchanges go to `inner` (the ranks actually running; None = this
    process alone).  Lets one GPU plan and time its share of an 8-GPU job."""

    def __init__(self, rank: int, world: int, gathers: list, inner: Comm | None = None):
        self.rank, self.world = rank, world
        self._gathers = list(gathers)
        self.inner = inner

    def all_gather_object(self, obj) -> list:
        out = list(self._gathers.pop(0))
        out[self.rank] = obj
        return out

    def all_reduce_sum_(self, tensor) -> None:
        if self.inner is not None:
            self.inner.all_reduce_sum_(tensor)

    def exchange(self, sends, recvs) -> None:
        if self.inner is not None:
            self.inner.exchange(sends, recvs)
        elif sends or recvs:
            raise N.NativeError("StaticComm: point-to-point traffic with ranks that are not running")


# ---------------------------------------------------------------------------
# record metadata that crosses ranks

@dataclass
class RecordMeta:
    """A trace record without its payload, plus where it lives."""

    id: object
    rank_meta: object
    mapping: object
    replica_group_size: int
    shape: tuple
    dtype_code: int
    module_class: str
    owner: int
    order: tuple
    record: object = None        # the local TraceRecord (None on other ranks)

    def __getstate__(self):
        state = dict(self.__dict__)
        state["record"] = None
        return state

    def device_payload(self):
        from .device import to_device
        if self.record is None:
            raise N.NativeError(f"{self.id.encode()}: payload lives on rank {self.owner}")
        return to_device(self.record.payload)


class _MetaTrace:
    def __init__(self, header: dict, records: list):
        self.header, self.records = header, records

    def by_id(self) -> dict:
        groups: dict = {}
        for k, rec in enumerate(self.records):
            groups.setdefault(rec.id.encode(), []).append((k, rec))
        return groups


def _metas(trace, rank: int, order_key) -> list:
    out = []
    for pos, rec in enumerate(trace.records):
        key = order_key(rec, pos) if order_key is not None else (rank, pos)
        out.append(RecordMeta(rec.id, rec.rank_meta, rec.mapping, rec.replica_group_size,
                              tuple(rec.shape), rec.dtype_code, rec.module_class, rank,
                              tuple(key) if isinstance(key, (tuple, list)) else (key,), rec))
    return out


def global_trace(trace, comm: Comm, order_key=None) -> _MetaTrace:
    """Every rank's record metadata, merged in global execution order
    (order_key(record, local position); default: rank-major)."""
    mine = _metas(trace, comm.rank, order_key)
    gathered = comm.all_gather_object(mine)
    allrecs = []
    for r, metas in enumerate(gathered):
        if r == comm.rank:
            allrecs.extend(mine)          # keep the local payload links
        else:
            allrecs.extend(metas)
    allrecs.sort(key=lambda m: m.order)
    return _MetaTrace(trace.header, allrecs)


# ---------------------------------------------------------------------------
# the distributed check

def allreduce_partials(prep, comm: Comm | None = None) -> None:
    """Sum the reduced slot vector of a Prepared plan across ranks, in place
    (NCCL enqueues on torch's current stream)."""
    import torch
    slots = prep.slot_sums
    if slots.numel() == 0:
        return
    if comm is None:
        import torch.distributed as dist
        with torch.cuda.stream(prep.stream):
            dist.all_reduce(slots, op=dist.ReduceOp.SUM)
        return
    with torch.cuda.stream(prep.stream):
        comm.all_reduce_sum_(slots)


class DistributedCheckPlan:
    """check() across ranks; construct and run collectively on every rank."""

    def __init__(self, ref, cand, tol, kappa: float = 3.0, *, fmt, comm: Comm, order_key=None):
        from .checker import CheckPlan, _require_same_setup
        from .errors import ConfigInvalid
        from .plan import Plan, PlanEntry, compare_copies, merge_view
        if kappa <= 0:
            raise ConfigInvalid("kappa must be positive")
        _require_same_setup(ref, cand)
        self.comm = comm
        self.ref, self.cand, self.tol, self.kappa, self.fmt = ref, cand, tol, kappa, fmt
        gref = global_trace(ref, comm, order_key)
        gcand = global_trace(cand, comm, order_key)
        self.ref_view = merge_view(gref)
        self.cand_view = merge_view(gcand)
        self.common = [i for i in self.cand_view if i in self.ref_view]
        self.plan = Plan([PlanEntry(i, x=self.ref_view[i], y=self.cand_view[i], x_rep=True,
                                    y_rep=True, tolerance=tol.get(i)) for i in self.common],
                         owner=lambda m: m.owner, me=comm.rank,
                         compare_copy=compare_copies(self.cand_view, lambda m: m.owner), digest=True)
        self._digest = None
        self.mode = str(cand.header.get("mode", ""))
        self._report = CheckPlan.report
        self._report_rows = lambda: CheckPlan._report_rows(self)

    def _remote_group_records(self, slot_entry):
        _, ei, side, gi = slot_entry
        e = self.plan.entries[ei]
        meta = e.y if side == 0 else e.x
        return meta.groups[gi].records

    def digests(self):
        """(table, Fingerprints, where, F): the digest table of this rank's
        copies of cross-rank replica groups.  Rows [0, F) are the digest
        slots td_segnorm fills while comparing (plan.fused_digests), rows
        [F, ...) the other local copies, digested by one td_fingerprint
        launch; where[row] = (remote group index, copy index).  Staged once;
        zero the table before each run."""
        if self._digest is None:
            import torch
            from .device import Fingerprints
            fused = list(self.plan.fused_digests)
            done = set(fused)
            where, tensors = list(fused), []
            for k, entry in enumerate(self.plan.remote_groups):
                for c, m in enumerate(self._remote_group_records(entry)):
                    if m.owner == self.comm.rank and (k, c) not in done:
                        where.append((k, c))
                        tensors.append(m.device_payload().reshape(-1))
            table = torch.zeros((max(len(where), 1), 2), dtype=torch.int64, device="cuda")
            fps = Fingerprints(tensors, out=table[len(fused):])
            self._digest = (table, fps, where, len(fused))
        return self._digest

    def _resolve_remote(self, table, where):
        """Exchange the digests (one all_reduce of a small table) and, on a
        mismatch (bug path only):
          * copy 0's rank receives the other copies and computes the exact
            replica sums — returned as {group slot: 8 sums} to add;
          * when the compare of that group reads a copy other than copy 0
            (compare_copies) and that copy differs from copy 0, its rank
            receives copy 0 and the compare must be re-run reading it —
            returned as {id(record): tensor} operand overrides.
        Messages are issued in remote-group order on every rank, so each
        (source, destination) pair sees sends and receives in the same order."""
        import torch
        from .device import _Raw, _one_group, resolve_operands
        from .plan import Plan, PlanEntry
        remote = self.plan.remote_groups
        if not remote:
            return {}, {}
        full = torch.zeros((len(remote), N.MAX_Z + 1, 2), dtype=torch.int64, device="cuda")
        if where:
            rows = torch.tensor([k for k, _ in where], device="cuda")
            cols = torch.tensor([c for _, c in where], device="cuda")
            full[rows, cols] = table[:len(where)]
        self.comm.all_reduce_sum_(full)
        fp = full.cpu().numpy()
        compare_copy = {(ei, gi): c for ei, gi, c in self.plan.compare_reads}
        me = self.comm.rank
        extra, overrides = {}, {}
        sends, recvs, pending = [], [], []
        for k, entry in enumerate(remote):
            recs = self._remote_group_records(entry)
            differs = [c for c in range(1, len(recs)) if not np.array_equal(fp[k, c], fp[k, 0])]
            if not differs:
                continue
            y0 = recs[0]
            if y0.owner == me:
                bufs = []
                for c, m in enumerate(recs[1:], start=1):
                    if m.owner == me:
                        bufs.append(m.device_payload().reshape(-1))
                    else:
                        buf = torch.empty(int(np.prod(m.shape)), dtype=_torch_dtype(m.dtype_code),
                                          device="cuda")
                        recvs.append((m.owner, buf))
                        bufs.append(buf)
                pending.append((entry[0], y0, bufs))
            else:
                for m in recs[1:]:
                    if m.owner == me:
                        sends.append((y0.owner, m.device_payload().reshape(-1)))
            _, ei, side, gi = entry
            cc = compare_copy.get((ei, gi), 0) if side == 0 else 0
            if cc and cc in differs:
                holder = recs[cc]
                if holder.owner == me and y0.owner == me:
                    overrides[id(holder)] = y0.device_payload()
                elif holder.owner == me:
                    buf = torch.empty(tuple(y0.shape), dtype=_torch_dtype(y0.dtype_code), device="cuda")
                    recvs.append((y0.owner, buf.view(-1)))
                    overrides[id(holder)] = buf
                elif y0.owner == me:
                    sends.append((holder.owner, y0.device_payload().reshape(-1)))
        self.comm.exchange(sends, recvs)
        for slot, y0, bufs in pending:
            raws = [_Raw(y0.device_payload().reshape(-1))] + [_Raw(b) for b in bufs]
            mini = Plan([PlanEntry("remote", x=None, y=_one_group("remote", raws, True),
                                   x_rep=False, y_rep=True)])
            ptrs, keep = resolve_operands(mini.operands, mini.operand_dtypes)
            sums: dict = {}
            mini.run(ptrs, sums=sums)
            extra[slot] = sums["group"][0]
        return extra, overrides

    def execute(self, timing: dict | None = None):
        """Digests of the local copies of cross-rank groups (td_fingerprint +
        the digest slots of the compare pass), td_segnorm, the digest
        exchange, then — only when a compare read a copy that differs from
        copy 0 — the compare pass again reading copy 0, slot reduction, the
        partial-sum all_reduce and the verdicts."""
        import torch
        from .device import resolve_operands
        table, fps, where, _ = self.digests()
        ptrs, keep = resolve_operands(self.plan.operands, self.plan.operand_dtypes)
        prep = self.plan.prepare(ptrs, kappa=self.kappa, eps=self.fmt.eps,
                                 replica_eps=self.fmt.eps, digests=table.data_ptr())
        sh = N.stream_handle(prep.stream)
        with torch.cuda.stream(prep.stream):
            table.zero_()
        # copies no local compare reads are digested beside the compare pass
        # (both stream HBM; each fills the other's tail)
        side = torch.cuda.Stream()
        side.wait_stream(prep.stream)
        fps.run(side)
        prep.segnorm(sh)
        prep.stream.wait_stream(side)
        extra, overrides = self._resolve_remote(table, where)
        if overrides:
            ptrs, keep2 = resolve_operands(self.plan.operands, self.plan.operand_dtypes, overrides)
            prep = self.plan.prepare(ptrs, kappa=self.kappa, eps=self.fmt.eps,
                                     replica_eps=self.fmt.eps, digests=table.data_ptr())
            sh = N.stream_handle(prep.stream)
            prep.segnorm(sh)
        prep.reduce(sh)
        if extra:
            gsum = prep.slot_sums[2 * prep.n_ids:].view(-1, N.SLOT_STRIDE)
            for slot, vals in extra.items():
                gsum[slot] += torch.from_numpy(vals).to(gsum.device)
        allreduce_partials(prep, self.comm)
        prep.verdict(sh)
        out = prep.fetch()
        del keep
        return out

    def run(self, timing: dict | None = None):
        idres, gres, ties = self.execute(timing)
        return self._report(self, idres, gres, ties)


def _torch_dtype(code: int):
    import torch
    return {N.F32: torch.float32, N.BF16: torch.bfloat16, N.F16: torch.float16,
            N.F64: torch.float64}[code]


def check_distributed(ref, cand, tol, kappa: float = 3.0, *, fmt, comm: Comm | None = None,
                      order_key=None):
    """Collective check(): each rank passes the records it holds.  Returns
    the full CheckReport on every rank."""
    comm = comm or TorchComm()
    return DistributedCheckPlan(ref, cand, tol, kappa, fmt=fmt, comm=comm,
                                order_key=order_key).run()


def split_reference(ref, cand_global, world: int):
    """Per-rank reference traces: each rank gets the reference slices that
    cover the global boxes of the candidate shards whose compare it runs
    (copy 0, or the copy plan.compare_copies picks for a cross-rank replica
    group), cut from the reference records it was given.

    cand_global: the candidate's global metadata trace (global_trace()), so
    owners are known.  Ids the candidate cannot merge, ids whose hulls
    differ, and reference-only ids keep their records whole on rank 0 (no
    compare runs for them)."""
    from .canonical import ShardMapping, SliceBox
    from .plan import compare_copies, merge_view
    from .tracestore import RankMeta, Trace, TraceRecord
    out = [Trace(header=ref.header, raw_header=ref.raw_header) for _ in range(world)]
    cview = merge_view(cand_global)
    rview = merge_view(ref)
    choice = compare_copies(cview, lambda m: m.owner)
    for ident, rmeta in rview.items():
        cmeta = cview.get(ident)
        records = [rec for g in rmeta.groups for rec in g.records]
        if (cmeta is None or not cmeta.merge_ok or not rmeta.merge_ok
                or cmeta.global_shape != rmeta.global_shape):
            out[0].records.extend(records)
            continue
        k = 0
        for gi, g in enumerate(cmeta.groups):
            y0 = g.records[choice.get((ident, gi), 0)]
            for _, gbox in y0.mapping.pairs:
                for rg in rmeta.groups:
                    x0 = rg.records[0]
                    for xl, xg in x0.mapping.pairs:
                        cut = []
                        for (a0, a1), (b0, b1) in zip(gbox.bounds, xg.bounds):
                            lo, hi = max(a0, b0), min(a1, b1)
                            if lo >= hi:
                                cut = None
                                break
                            cut.append((lo, hi))
                        if cut is None:
                            continue
                        ext = tuple(hi - lo for lo, hi in cut)
                        src = tuple(slice(l0 + c0 - g0, l0 + c0 - g0 + e)
                                    for (l0, _), (g0, _), (c0, _), e in zip(xl.bounds, xg.bounds, cut, ext))
                        payload = x0.payload[src]
                        payload = payload.contiguous() if hasattr(payload, "contiguous") else \
                            np.ascontiguousarray(payload)
                        local = SliceBox(tuple((0, e) for e in ext))
                        mapping = ShardMapping(ext, rmeta.global_shape, ((local, SliceBox(tuple(cut))),))
                        piece = TraceRecord(x0.id, RankMeta(0, k, 0, 0, 0, 0), mapping, 1, payload,
                                            x0.module_class)
                        piece.parent = getattr(x0, "record", None) or x0
                        out[y0.owner].records.append(piece)
                        k += 1
    return out
