"""Host planner + executor of the compare hot path.

Planning is metadata only.  For each canonical id it reproduces
checker._merge_one (pkg/src/traindiff/checker.py:151-198) up to the
arithmetic: rank agreement, per-axis hull, grouping of records by
(local shape, pairs), the declared replica-group size, mapping validation
and the merge witnesses (data-free, see canonical.py).  It then lays the
arithmetic out as *segments* — 2-D strided blocks read in lockstep from the
reference side (x), candidate copy 0 (y) and the candidate's replica copies
(z) — cut from the intersections of candidate and reference global boxes, so
the merged tensors are never materialised and every payload byte is read
once.  Segments are split into fixed-size tiles; one persistent kernel per
tile class (dtype x replica count) walks them (td_segnorm), then
td_reduce_slots and td_verdict turn tile partials into per-id verdicts.

A `Plan` captures structure only: it holds (record, byte offset) for every
operand and patches device addresses in at `run()` time, so a plan built
once for a layout can be re-run on every step's fresh payloads.
"""

from __future__ import annotations

import contextlib
import functools
import gc
import itertools
import math
import os
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .canonical import ShardMapping, merge_problem

# per-structure templates in merge_view and Plan (TD_PLAN_TEMPLATES=0: the
# general path for every id; tests/test_plan_templates.py checks they agree)
_TEMPLATES = os.environ.get("TD_PLAN_TEMPLATES", "1") != "0"

VERDICT_NAMES = {N.PASS: "pass", N.FLAG: "flag", N.REPLICA: "replica-mismatch",
                 N.MERGE: "merge-error", N.MISSING: "missing"}
MAX_UNITS = 1 << 30          # per-segment unit cap (kernel uses 32-bit unit indices)
_VEC_DTYPES = (N.F32, N.BF16, N.F16)

# column layout of a plan's segment rows once frozen to int64 (Plan._columns):
# x slot (-1: none), x offset, y slot, y offset, MAX_Z z slots (-1 padded),
# nz, rows, cols, x row stride, y row stride, first tile, units, vector flag,
# digest slot (-1: none); offsets / strides in elements
_C_X, _C_XO, _C_Y, _C_YO, _C_Z = 0, 1, 2, 3, 4
_C_NZ = _C_Z + N.MAX_Z
_C_R, _C_C, _C_RX, _C_RY, _C_TB, _C_NU, _C_VEC, _C_DS = range(_C_NZ + 1, _C_NZ + 9)
_TPL_NCOLS = _C_DS + 1
_SLOT_COLS = [_C_X, _C_Y] + list(range(_C_Z, _C_Z + N.MAX_Z))
_ESIZE = np.zeros(max(N.DTYPE_SIZE) + 1, np.int64)
for _code, _size in N.DTYPE_SIZE.items():
    _ESIZE[_code] = _size


@contextlib.contextmanager
def no_gc():
    """Cyclic GC paused while a plan is built: planning allocates tens of
    thousands of small tuples, and a full collection over a process holding
    big traces (every record, every payload handle) costs more than the
    planning itself (config 2: 131 ms vs 28 ms for the segment tables).
    Nothing built here is cyclic garbage; reference counting frees it."""
    if not gc.isenabled():
        yield
        return
    gc.disable()
    try:
        yield
    finally:
        gc.enable()


def gc_paused(fn):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        with no_gc():
            return fn(*args, **kwargs)
    return wrapper


# ---------------------------------------------------------------------------
# merge metadata (checker.py:151-198 without the arithmetic)

@dataclass
class GroupMeta:
    records: list                 # copies of one shard, record order
    declared_detail: str | None   # replica-size declaration problem, if any
    numeric: bool                 # copies need the device rel_err check


class IdMeta:
    """Merge metadata of one id: its shard groups (copies of one shard) and
    problems.  merge_view's template path leaves `groups` lazy — (trace
    records, the id's record positions, the structure's group template) —
    until something reads them: the planner's replay takes records straight
    from the template (record_at) and only problem ids are ever detailed."""

    __slots__ = ("ident", "exec_index", "global_shape", "rank_problem", "merge_detail", "struct_key",
                 "_groups", "_lazy")

    def __init__(self, ident: str, exec_index: int, groups: list | None = None,
                 global_shape: tuple | None = None, rank_problem: bool = False,
                 merge_detail: str | None = None, struct_key: int | None = None):
        self.ident, self.exec_index = ident, exec_index
        self.global_shape, self.rank_problem, self.merge_detail = global_shape, rank_problem, merge_detail
        self.struct_key = struct_key          # interned merge_view structure (copy signatures, sizes, dtypes)
        self._groups = [] if groups is None else groups
        self._lazy = None                     # (records, positions, [(idx, declared detail, numeric)])

    @property
    def groups(self) -> list:
        lazy = self._lazy
        if lazy is not None:
            recs, ks, tgroups = lazy
            self._groups = [GroupMeta(records=[None if recs is None else recs[ks[k]] for k in idx],
                                      declared_detail=d, numeric=num) for idx, d, num in tgroups]
            self._lazy = None
        return self._groups

    @groups.setter
    def groups(self, value: list) -> None:
        self._groups, self._lazy = value, None

    def record_at(self, gi: int, ri: int):
        """groups[gi].records[ri] without materialising the groups."""
        lazy = self._lazy
        if lazy is None:
            return self._groups[gi].records[ri]
        recs, ks, tgroups = lazy
        return recs[ks[tgroups[gi][0][ri]]]

    def all_records(self):
        """Every record of the id's groups (any order)."""
        lazy = self._lazy
        if lazy is not None and lazy[0] is not None:
            recs = lazy[0]
            return [recs[k] for k in lazy[1]]
        return itertools.chain.from_iterable(g.records for g in self._groups)

    def drop_records(self) -> None:
        """Forget the trace's records (cached plans keep metadata only)."""
        if self._lazy is not None:
            self._lazy = (None, self._lazy[1], self._lazy[2])
        else:
            for g in self._groups:
                g.records = [None] * len(g.records)

    @property
    def merge_ok(self) -> bool:
        return not self.rank_problem and self.merge_detail is None

    @property
    def declared_problem(self) -> str | None:
        if self._lazy is not None:
            for _, d, _ in self._lazy[2]:
                if d is not None:
                    return d
            return None
        for g in self._groups:
            if g.declared_detail is not None:
                return g.declared_detail
        return None

    def __repr__(self) -> str:
        return (f"IdMeta(ident={self.ident!r}, exec_index={self.exec_index}, global_shape={self.global_shape}, "
                f"groups={len(self.groups)})")


def id_meta(ident: str, entries: list, replica_check: bool = True) -> IdMeta:
    """entries: [(exec index, TraceRecord)] sorted by exec index."""
    meta = IdMeta(ident=ident, exec_index=entries[0][0])
    ranks = {len(rec.mapping.global_shape) for _, rec in entries}
    if len(ranks) != 1:
        meta.rank_problem = True
        meta.merge_detail = "records disagree on tensor rank"
        return meta
    (ndim,) = ranks
    hull = tuple(max(rec.mapping.global_shape[a] for _, rec in entries) for a in range(ndim))
    meta.global_shape = hull
    buckets: dict[tuple, list] = {}
    for _, rec in entries:
        key = (rec.mapping.local_shape, rec.mapping.pairs_bounds)
        buckets.setdefault(key, []).append(rec)
    for recs in buckets.values():
        detail = None
        numeric = False
        if replica_check:
            declared = {rec.replica_group_size for rec in recs}
            if declared != {len(recs)}:
                detail = (f"{len(recs)} copies of one shard, declared replica group size "
                          f"{sorted(declared)}")
            else:
                numeric = len(recs) > 1
        meta.groups.append(GroupMeta(records=recs, declared_detail=detail, numeric=numeric))
    maps = tuple(g.records[0].mapping for g in meta.groups)
    shapes = tuple(tuple(g.records[0].shape) for g in meta.groups)
    key = (tuple(m.signature() for m in maps), hull, shapes)
    detail = _MERGE_DETAIL.get(key, _MISSING)
    if detail is _MISSING:
        if len(_MERGE_DETAIL) > 65536:
            _MERGE_DETAIL.clear()
        detail = _MERGE_DETAIL[key] = _merge_detail(maps, hull, shapes)
    meta.merge_detail = detail
    return meta


_MERGE_DETAIL: dict = {}
_MISSING = object()


def _merge_detail(mappings: tuple, hull: tuple, shapes: tuple) -> str | None:
    """merge()'s verdict for these shard layouts, memoised by the layouts'
    signatures (id_meta): every id of one layout (all hidden activations,
    say) shares one validation."""
    normed = [ShardMapping(m.local_shape, hull, m.pairs) for m in mappings]
    err = merge_problem(normed, hull, list(shapes))
    return None if err is None else str(err)


@gc_paused
def merge_view(trace, replica_check: bool = True) -> dict[str, IdMeta]:
    """Per-id merge metadata in first-appearance order (checker.py:201-211).

    id_meta reads only each record's mapping and declared replica size, so
    ids whose records carry the same (mapping signature, replica size)
    sequence share one result shape: it is computed once per structure and
    re-instantiated with each id's own records (`_TEMPLATES`)."""
    from .tracestore import Trace
    ext = N.host_ext()
    if _TEMPLATES and ext is not None and type(trace).by_id is Trace.by_id:
        recs = list(trace.records)       # the lazy metas resolve positions against this snapshot
        return _merge_view_grouped(recs, ext.group_by_id(recs), replica_check)
    view = {}
    memo: dict | None = {} if _TEMPLATES else None
    for ident, entries in trace.by_id().items():
        # by_id lists an id's records in trace order: already sorted by position
        if memo is None:
            view[ident] = id_meta(ident, entries, replica_check)
            continue
        key = tuple((rec.mapping.sig_id, rec.replica_group_size, rec.dtype_code) for _, rec in entries)
        hit = memo.get(key)
        if hit is None:
            meta = view[ident] = id_meta(ident, entries, replica_check)
            pos = {id(rec): k for k, (_, rec) in enumerate(entries)}
            if len(pos) != len(entries):         # one record object listed twice: no template
                continue
            # the groups are a function of `key`, which also holds the copies'
            # dtypes: everything the per-entry planner reads (plan templates);
            # interned to a small int so entry keys hash cheaply
            hit = memo[key] = (meta.rank_problem, meta.global_shape, meta.merge_detail,
                               [([pos[id(r)] for r in g.records], g.declared_detail, g.numeric)
                                for g in meta.groups], _intern_struct((replica_check, key)))
        else:
            rank_problem, hull, detail, groups, _ = hit
            meta = view[ident] = IdMeta(ident=ident, exec_index=entries[0][0], global_shape=hull,
                                        rank_problem=rank_problem, merge_detail=detail)
            meta.groups = [GroupMeta(records=[entries[k][1] for k in idx], declared_detail=d, numeric=num)
                           for idx, d, num in groups]
        meta.struct_key = hit[4]
    return view


def _merge_view_grouped(recs: list, grouped, replica_check: bool) -> dict[str, IdMeta]:
    """merge_view's template path over _td_host.group_by_id's output (ids in
    first-appearance order, their record positions, their structure keys):
    the same metadata, without the per-record Python walks; ids that repeat
    a structure keep their groups lazy (IdMeta.groups)."""
    view = {}
    memo: dict = {}
    for ident, ks, key in zip(*grouped):
        hit = memo.get(key)
        if hit is None:
            entries = [(k, recs[k]) for k in ks]
            meta = view[ident] = id_meta(ident, entries, replica_check)
            pos = {id(rec): k for k, (_, rec) in enumerate(entries)}
            if len(pos) != len(entries):         # one record object listed twice: no template
                continue
            hit = memo[key] = (meta.rank_problem, meta.global_shape, meta.merge_detail,
                               [([pos[id(r)] for r in g.records], g.declared_detail, g.numeric)
                                for g in meta.groups], _intern_struct((replica_check, key)))
        else:
            rank_problem, hull, detail, groups, _ = hit
            meta = view[ident] = IdMeta(ident=ident, exec_index=ks[0], global_shape=hull,
                                        rank_problem=rank_problem, merge_detail=detail)
            meta._lazy = (recs, ks, groups)
        meta.struct_key = hit[4]
    return view


# ---------------------------------------------------------------------------
# segment construction

def _magic(d: int) -> tuple[int, int]:
    """(m, p) with floor(n / d) == (n * m) >> p for 0 <= n < 2^31."""
    l = (d - 1).bit_length()
    p = 31 + l
    return (1 << p) // d + (1 if (1 << p) % d else 0), p


def _strides(shape: tuple) -> list[int]:
    out, acc = [0] * len(shape), 1
    for a in range(len(shape) - 1, -1, -1):
        out[a] = acc
        acc *= shape[a]
    return out


def _blocks(ext, x_start, x_shape, y_start, y_shape):
    """Decompose an N-d box (extents `ext`) read at x_start in an array of
    x_shape and at y_start in y_shape into 2-D strided blocks:
    yields (x_off, y_off, rows, cols, x_row_stride, y_row_stride) in elements."""
    d = len(ext)
    if any(e == 0 for e in ext):
        return
    if d == 0:
        yield 0, 0, 1, 1, 1, 1
        return
    xs, ys = _strides(x_shape), _strides(y_shape)
    k = d - 1
    while k > 0 and ext[k] == x_shape[k] and ext[k] == y_shape[k]:
        k -= 1
    cols = math.prod(ext[k:])
    if k == 0:
        rows, rx, ry, outer = 1, cols, cols, []
    else:
        rows, rx, ry, outer = ext[k - 1], xs[k - 1], ys[k - 1], list(range(k - 1))
    base_x = sum(x_start[a] * xs[a] for a in range(d) if a not in outer)
    base_y = sum(y_start[a] * ys[a] for a in range(d) if a not in outer)
    for combo in np.ndindex(*[ext[a] for a in outer]) if outer else [()]:
        ox = base_x + sum((x_start[a] + i) * xs[a] for a, i in zip(outer, combo))
        oy = base_y + sum((y_start[a] + i) * ys[a] for a, i in zip(outer, combo))
        yield ox, oy, rows, cols, rx, ry


class _Operand:
    """A registered payload: slot in the plan's operand table, the dtype it
    is read as, that dtype's size."""

    __slots__ = ("slot", "dtype", "esize")

    def __init__(self, slot: int, dtype: int, esize: int):
        self.slot, self.dtype, self.esize = slot, dtype, esize


class PlanBuilder:
    """Accumulates segments; operands are registered payloads (records)."""

    def __init__(self, force_generic: bool = False):
        self.force_generic = force_generic
        self.operands: list = []          # payload owners (records or raw tensors)
        self.operand_dtypes: list = []    # dtype each operand is read as
        self._operand_index: dict = {}
        self.seg_rows: list = []          # (xs, xoff, ys, yoff, zs, rows, cols, rx, ry, tile_begin, n_units, vec_ok,
        #                                    digest slot or -1)
        self.n_tiles = 0
        self.digest_slot = -1             # stamped on segments emitted while >= 0
        self.classes: dict = {}           # class key -> list of (tile_begin, n_tiles)

    def operand(self, owner, dtype: int) -> _Operand:
        """Register `owner`'s payload, to be presented to the kernel as `dtype`
        (a widening cast at resolution time when the stored dtype differs)."""
        key = (id(owner), dtype)
        op = self._operand_index.get(key)
        if op is None:
            op = _Operand(len(self.operands), dtype, N.DTYPE_SIZE[dtype])
            self.operands.append(owner)
            self.operand_dtypes.append(dtype)
            self._operand_index[key] = op
        return op

    def add(self, x: _Operand | None, x_off: int, y: _Operand, y_off: int, zs: list,
            rows: int, cols: int, rx: int, ry: int) -> None:
        if rows == 0 or cols == 0:
            return
        same = [y.dtype] + [z.dtype for z in zs] + ([x.dtype] if x is not None else [])
        vec_dtype = (not self.force_generic and same[0] in _VEC_DTYPES
                     and all(d == same[0] for d in same))
        if rows == 1 and vec_dtype and cols > 8 and cols % 8:
            # a flat run whose length is not a multiple of the vector (an odd
            # vocabulary, say): vector head, element-wise tail of < 8 cells
            head = cols - cols % 8
            self.add(x, x_off, y, y_off, zs, 1, head, rx, ry)
            self.add(x, x_off + head, y, y_off + head, zs, 1, cols - head, rx, ry)
            return
        esize = y.esize
        # row-stride alignment is a property of the layout; base alignment is
        # re-checked against live addresses at run time
        vec = (vec_dtype and cols % 8 == 0
               and (rows == 1 or ((ry * esize) % 16 == 0
                                  and (x is None or (rx * x.esize) % 16 == 0)))
               and (x_off * (x.esize if x else 0)) % 16 == 0 and (y_off * esize) % 16 == 0)
        unit = 8 if vec else 1
        upr = cols // unit
        if rows == 1:
            step = max(unit, (MAX_UNITS // 1) * unit)
            for c0 in range(0, cols, step):
                cc = min(step, cols - c0)
                self._emit(x, x_off + c0, y, y_off + c0, zs, 1, cc, rx, ry, vec)
            return
        rows_per = max(1, MAX_UNITS // max(upr, 1))
        if upr > MAX_UNITS:
            for r in range(rows):
                self.add(x, x_off + r * rx, y, y_off + r * ry, zs, 1, cols, rx, ry)
            return
        for r0 in range(0, rows, rows_per):
            rr = min(rows_per, rows - r0)
            self._emit(x, x_off + r0 * rx, y, y_off + r0 * ry, zs, rr, cols, rx, ry, vec)

    def _emit(self, x, x_off, y, y_off, zs, rows, cols, rx, ry, vec):
        unit = 8 if vec else 1
        n_units = rows * cols // unit
        n_tiles = -(-n_units // N.TILE_UNITS)
        self.seg_rows.append((x, x_off, y, y_off, list(zs), rows, cols, rx, ry,
                              self.n_tiles, n_units, vec, self.digest_slot))
        self.n_tiles += n_tiles

    @property
    def tile_cursor(self) -> int:
        return self.n_tiles


# ---------------------------------------------------------------------------
# plans

def compare_copies(view: dict, owner) -> dict:
    """Which copy of each cross-rank replica group the representative compare
    reads (multi-GPU): {(ident, group index): copy index}.

    The reference compares copy 0 of every shard group (checker.py:184-191).
    When the copies of a replica-checked group live on several ranks they are
    all digested (td_fingerprint) where they live, and equal digests mean
    every copy IS copy 0 — so the compare may read whichever copy is least
    loaded instead of always copy 0's rank (which, for DP-replicated
    parameters and TP-replicated activations, would pile every compare on the
    dp=0 / tp=0 GPUs: 1.6x the mean on config 4).  Greedy, largest group
    first, onto the holder with the fewest bytes to read so far; ties keep
    the lower copy index.  Deterministic from the global view, so every rank
    and split_reference agree.  On a digest mismatch (bug path) the compare
    holder is handed copy 0 (distributed.py) so the result stays exact."""
    load: dict = {}
    remote = []
    for ident, meta in view.items():
        if meta.rank_problem:
            continue
        for gi, g in enumerate(meta.groups):
            recs = g.records
            nb = math.prod(recs[0].shape) * N.DTYPE_SIZE[recs[0].dtype_code]
            owners = [owner(r) for r in recs]
            for o in owners:
                load[o] = load.get(o, 0) + nb          # digest / fused replica read
            if g.numeric and len(set(owners)) > 1:
                remote.append((nb, ident, gi, owners))
            else:
                load[owners[0]] = load.get(owners[0], 0) + nb   # the reference slice
    remote.sort(key=lambda t: -t[0])
    out = {}
    for nb, ident, gi, owners in remote:
        best = min(range(len(owners)), key=lambda c: (load[owners[c]], c))
        out[(ident, gi)] = best
        load[owners[best]] += 2 * nb                   # copy re-read + reference slice
    return out


@dataclass
class PlanEntry:
    ident: str
    x: IdMeta | None          # reference side (or base in tolerance estimation)
    y: IdMeta | None          # candidate side
    x_rep: bool               # run numeric replica checks on x's groups
    y_rep: bool
    tolerance: float = 0.0


class Plan:
    """Frozen layout of one comparison; `run()` executes it on the GPU."""

    @gc_paused
    def __init__(self, entries: list[PlanEntry], static: tuple[float, float] | None = None,
                 owner=None, me: int = 0, compare_copy: dict | None = None, digest: bool = False,
                 disjoint: bool = False):
        """static=(atol, rtol) builds compare_static's plan: the elementwise
        failure count replaces d2 (generic walker, no replica checks).

        owner(record) -> rank restricts the plan to the records rank `me`
        holds (multi-GPU, distributed.py).  Id and replica-group slots are
        laid out identically on every rank; a rank emits segments only for
        work whose operands it holds: compare runs on the rank holding the
        candidate's copy 0 (the reference slice must be there too), fused
        replica sums when every copy of the group is on that rank.  Groups
        whose copies span ranks are listed in `remote_groups` and resolved
        by fingerprints (zero sums = identical copies).  compare_copy
        (compare_copies()) picks which copy of such a group the compare
        reads; `compare_reads` lists (entry, group index, copy index) for
        the groups where it is not copy 0.  digest=True digests the copy a
        local compare of a cross-rank group reads inside that compare
        (td_segnorm digest classes) when its segments cover the record
        exactly once; `fused_digests` lists (remote group index, copy index)
        per digest slot, the other local copies still need td_fingerprint."""
        self.entries = entries
        self.static = static
        owner_given = owner
        owner = owner if owner is not None else (lambda rec: me)
        is_local = (lambda rec: owner(rec) == me)
        b = PlanBuilder(force_generic=static is not None)
        id_rows = []
        group_rows = []
        self._group_owner = []     # (entry index, side, group index) per group slot
        self.group_offset = []    # per group slot: copy index of its first replica - 1
        self.subslots = {}        # first group slot -> all slots of that group (> MAX_Z + 1 copies)
        self.remote_groups = []   # (first group slot, entry index, side, group index)
        self.compare_reads = []   # (entry index, group index, copy index != 0)
        self.fused_digests = []   # digest slot -> (remote group index, copy index)
        compare_copy = compare_copy or {}
        # per-entry templates (single-GPU plans): ids of one layout repeat a
        # few structures (every hidden activation, every weight of a shape);
        # the first id of a structure is planned in full and its output
        # recorded relative to its own operands / tiles / group slots, later
        # ids of the same structure replay it with their own records
        templates = {} if _TEMPLATES else None
        self._tpl_rows = []       # template k -> its segment rows (int64, _TPL_COLS)
        self._tpl_groups = []     # template k -> its group rows (tile begin, tile end relative; nz)
        self._tpl_ids = []        # template k -> its id row, relative
        self._replays = []        # (template, first operand, first tile, digest base, first group slot,
        #                            id row) per replayed entry
        self._id_tol = []         # tolerance per replayed entry, replay order
        self._owner_fill = []     # (first group slot, entry, ((side, group index), ...)) per replay
        # disjoint: the caller knows the two sides hold no record in common
        shared = _shared_entries(entries) if templates is not None and not disjoint else set()
        for ei, e in enumerate(entries):
            if templates is None:
                self._plan_entry(b, ei, e, group_rows, id_rows, owner, is_local, compare_copy, digest, static)
                continue
            key = None if ei in shared else (e.x_rep, e.y_rep, _meta_key(e.x), _meta_key(e.y))
            if key is not None and owner_given is not None:
                # multi-GPU plans also depend on where every copy lives and on
                # which copy each cross-rank group's compare reads
                key = (key, _owners_key(e.y, owner), _owners_key(e.x, owner),
                       tuple(compare_copy.get((e.ident, gi), 0) for gi in range(len(e.y.groups)))
                       if compare_copy and e.y is not None else ())
            tpl = templates.get(key) if key is not None else None
            if tpl is not None:
                self._replay_entry(b, ei, e, tpl, group_rows, id_rows)
                continue
            mark = (len(b.operands), len(b.seg_rows), b.n_tiles, len(group_rows), len(self._group_owner),
                    len(self.remote_groups), len(self.compare_reads), len(self.fused_digests))
            self._plan_entry(b, ei, e, group_rows, id_rows, owner, is_local, compare_copy, digest, static)
            if key is not None:
                templates[key] = self._record_entry(b, e, mark, group_rows, id_rows)
        self.builder = b
        self.n_tiles = b.n_tiles
        self._fill_replayed_rows(id_rows, group_rows)
        self._columns()
        self.tile_shift = self._retile()
        self._freeze_segments()
        del self._cols, self._replays, self._tpl_rows, self._tpl_groups, self._tpl_ids, self._id_tol
        self._chunk_slots()

    def _plan_entry(self, b: PlanBuilder, ei: int, e: PlanEntry, group_rows: list, id_rows: list, owner,
                    is_local, compare_copy: dict, digest: bool, static) -> None:
        """Segments, group slots and the id row of one entry (the general path)."""
        t0 = b.tile_cursor
        has_compare = (e.x is not None and e.y is not None and e.x.merge_ok and e.y.merge_ok
                       and e.x.global_shape == e.y.global_shape)
        cg0 = len(group_rows)
        if e.y is not None and not e.y.rank_problem:
            for gi, g in enumerate(e.y.groups):
                rep = e.y_rep and g.numeric
                s0 = b.tile_cursor
                y0 = g.records[0]
                spans = rep and len({owner(r) for r in g.records}) > 1
                c = 0
                if spans:
                    self.remote_groups.append((len(group_rows), ei, 0, gi))
                    c = compare_copy.get((e.ident, gi), 0)
                    if c:
                        y0 = g.records[c]
                        self.compare_reads.append((ei, gi, c))
                mine = is_local(y0)
                together = rep and not spans and mine
                # replica copies in chunks of MAX_Z (one group slot each);
                # the compare reads copy 0 with the first chunk, every
                # further chunk re-reads copy 0 once
                chunks = _replica_chunks(len(g.records)) if rep else []
                zall = []
                if mine:
                    gdt = _group_dtype(g.records) if together else y0.dtype_code
                    yop = b.operand(y0, gdt)
                    zall = [b.operand(r, gdt) for r in g.records[1:]] if together else []
                    zops = zall[:N.MAX_Z]
                    if has_compare:
                        fuse = digest and spans and static is None
                        first_seg = len(b.seg_rows)
                        if fuse:
                            b.digest_slot = len(self.fused_digests)
                        self._compare_runs(b, e.x, y0, yop, zops, is_local)
                        b.digest_slot = -1
                        if fuse:
                            self._settle_digest(b, first_seg, y0, yop, len(self.remote_groups) - 1, c)
                        if zops:
                            self._replica_remainder(b, y0, yop, zops)
                    elif zops:
                        n = math.prod(y0.shape)
                        b.add(None, 0, yop, 0, zops, 1, n, n, n)
                if rep:
                    self._group_slots(b, group_rows, chunks, s0, yop if zall else None, zall,
                                      math.prod(y0.shape), (ei, 0, gi))
        cg1 = len(group_rows)
        rg0 = len(group_rows)
        if e.x is not None and e.x_rep and not e.x.rank_problem:
            for gi, g in enumerate(e.x.groups):
                if not g.numeric:
                    continue
                s0 = b.tile_cursor
                x0 = g.records[0]
                mine = is_local(x0)
                chunks = _replica_chunks(len(g.records))
                zall, yop = [], None
                n = math.prod(x0.shape)
                if len({owner(r) for r in g.records}) > 1:
                    self.remote_groups.append((len(group_rows), ei, 1, gi))
                elif mine:
                    gdt = _group_dtype(g.records)
                    yop = b.operand(x0, gdt)
                    zall = [b.operand(r, gdt) for r in g.records[1:]]
                    b.add(None, 0, yop, 0, zall[:N.MAX_Z], 1, n, n, n)
                self._group_slots(b, group_rows, chunks, s0, yop, zall, n, (ei, 1, gi))
        rg1 = len(group_rows)
        cand_host = 0
        if e.y is not None:
            if e.y.declared_problem is not None:
                cand_host = N.REPLICA
            elif not e.y.merge_ok:
                cand_host = N.MERGE
        ref_host = 0
        if e.x is not None:
            if e.x.declared_problem is not None:
                ref_host = N.REPLICA
            elif not e.x.merge_ok:
                ref_host = N.MERGE
        id_rows.append((t0, b.tile_cursor, cg0, cg1, rg0, rg1, int(has_compare),
                        cand_host, ref_host, 0, float(e.tolerance)))

    def _record_entry(self, b: PlanBuilder, e: PlanEntry, mark: tuple, group_rows: list, id_rows: list):
        """The output of the entry just planned, relative to where it started
        (None when it cannot be replayed: an operand shared with another
        entry)."""
        n_ops, n_rows, tiles0, g0, o0, rg0_, cr0, fd0 = mark
        role = {}
        for side, meta in ((0, e.y), (1, e.x)):
            if meta is None:
                continue
            for gi, g in enumerate(meta.groups):
                for ri, r in enumerate(g.records):
                    role[id(r)] = (side, gi, ri)
        ops = []
        for owner_rec, dt in zip(b.operands[n_ops:], b.operand_dtypes[n_ops:]):
            where = role.get(id(owner_rec))
            if where is None:
                return None
            ops.append((where, dt))

        def rel(op):
            k = op.slot - n_ops
            if k < 0:
                raise LookupError
            return k
        try:
            # one int64 row per segment (_TPL_COLS), operand slots / tiles /
            # digest slots relative to the entry's start: replayed column-wise
            # for every later id of the structure in _columns()
            rows = np.array([(-1 if x is None else rel(x), xo, rel(y), yo,
                              *[rel(z) for z in zs], *([-1] * (N.MAX_Z - len(zs))), len(zs),
                              r, c, rx, ry, tb - tiles0, nu, int(vec), ds if ds < 0 else ds - fd0)
                             for x, xo, y, yo, zs, r, c, rx, ry, tb, nu, vec, ds in b.seg_rows[n_rows:]],
                            np.int64).reshape(-1, _TPL_NCOLS)
        except LookupError:
            return None
        remote = [(slot - g0, side, gi) for slot, _, side, gi in self.remote_groups[rg0_:]]
        reads = [(gi, c) for _, gi, c in self.compare_reads[cr0:]]
        fused = [(k - rg0_, c) for k, c in self.fused_digests[fd0:]]
        groups = [(s0 - tiles0, s1 - tiles0, nz) for s0, s1, nz in group_rows[g0:]]
        owners = [(side, gi) for _, side, gi in self._group_owner[o0:]]
        offsets = self.group_offset[o0:]
        subs = {k - g0: [j - g0 for j in v] for k, v in self.subslots.items() if k >= g0}
        t0, t1, cg0, cg1, rg0, rg1, hc, ch, rh, pad, _ = id_rows[-1]
        idrow = (t0 - tiles0, t1 - tiles0, cg0 - g0, cg1 - g0, rg0 - g0, rg1 - g0, hc, ch, rh, pad)
        self._tpl_rows.append(rows)
        self._tpl_groups.append(np.array(groups, np.int64).reshape(-1, 3))
        self._tpl_ids.append(idrow)
        return (tuple(w for w, _ in ops), tuple(dt for _, dt in ops), len(self._tpl_rows) - 1,
                b.n_tiles - tiles0, (None,) * len(groups), tuple(owners), offsets, subs, remote, reads, fused)

    def _replay_entry(self, b: PlanBuilder, ei: int, e: PlanEntry, tpl, group_rows: list, id_rows: list) -> None:
        where, dts, tpl_k, n_tiles, holes, owners, offsets, subs, remote, reads, fused = tpl
        fd0, rg0 = len(self.fused_digests), len(self.remote_groups)
        sides = (e.y, e.x)
        # a replayed entry's records are its own (shared records take the
        # general path, _shared_entries), so its operands need no
        # de-duplication entry: they are appended as one block
        op0 = len(b.operands)
        b.operands.extend([sides[side].record_at(gi, ri) for side, gi, ri in where])
        b.operand_dtypes.extend(dts)
        tiles0, g0 = b.n_tiles, len(group_rows)
        # segments, group rows and the id row are instantiated column-wise
        # later (_columns, _fill_replayed_rows); here only their slots
        self._replays.append((tpl_k, op0, tiles0, fd0, g0, len(id_rows)))
        if remote:
            self.remote_groups.extend((g0 + slot, ei, side, gi) for slot, side, gi in remote)
            self.compare_reads.extend((ei, gi, c) for gi, c in reads)
            self.fused_digests.extend((rg0 + k, c) for k, c in fused)
        b.n_tiles += n_tiles
        if holes:
            group_rows.extend(holes)
            self._group_owner.extend(holes)           # (ei, side, gi) filled on demand (_owners)
            self._owner_fill.append((g0, ei, owners))
            self.group_offset.extend(offsets)
            for k, v in subs.items():
                self.subslots[g0 + k] = [g0 + j for j in v]
        id_rows.append(None)
        self._id_tol.append(e.tolerance)

    _GROUP_DT = [("tile_begin", "<i8"), ("tile_end", "<i8"), ("nz", "<i4")]

    def _fill_replayed_rows(self, id_rows: list, group_rows: list) -> None:
        """self.ids / self.groups: the general path's rows as built, every
        replayed entry's rows from its template, offset column-wise by the
        entry's first tile / first group slot (per template, all replays at
        once)."""
        ids = np.zeros(len(id_rows), N.ID_DESC)
        groups = np.zeros(len(group_rows), self._GROUP_DT)
        gen_ids = [k for k, r in enumerate(id_rows) if r is not None]
        if gen_ids:
            ids[gen_ids] = np.array([id_rows[k] for k in gen_ids], N.ID_DESC)
        gen_groups = [k for k, r in enumerate(group_rows) if r is not None]
        if gen_groups:
            groups[gen_groups] = np.array([group_rows[k] for k in gen_groups], self._GROUP_DT)
        if self._replays:
            rp = np.array(self._replays, np.int64)   # template, op0, tiles0, fd0, g0, id row
            tol = np.array(self._id_tol, np.float64)
            order = np.argsort(rp[:, 0], kind="stable")
            for sel in np.split(order, np.flatnonzero(np.diff(rp[order, 0])) + 1):
                k = int(rp[sel[0], 0])
                t0, t1, cg0, cg1, rg0, rg1, hc, ch, rh, pad = self._tpl_ids[k]
                tiles0, g0, row = rp[sel, 2], rp[sel, 4], rp[sel, 5]
                ids["tile_begin"][row], ids["tile_end"][row] = tiles0 + t0, tiles0 + t1
                ids["cgroup_begin"][row], ids["cgroup_end"][row] = g0 + cg0, g0 + cg1
                ids["rgroup_begin"][row], ids["rgroup_end"][row] = g0 + rg0, g0 + rg1
                ids["has_compare"][row], ids["cand_host"][row], ids["ref_host"][row] = hc, ch, rh
                ids["pad"][row] = pad
                ids["tolerance"][row] = tol[sel]
                G = self._tpl_groups[k]
                if len(G):
                    slots = (g0[:, None] + np.arange(len(G))).reshape(-1)
                    groups["tile_begin"][slots] = (tiles0[:, None] + G[:, 0]).reshape(-1)
                    groups["tile_end"][slots] = (tiles0[:, None] + G[:, 1]).reshape(-1)
                    groups["nz"][slots] = np.tile(G[:, 2], len(sel))
        self.ids, self.groups = ids, groups

    @property
    def group_owner(self) -> list:
        """(entry index, side, group index) per group slot."""
        self._owners()
        return self._group_owner

    def _owners(self) -> None:
        """Fill the (entry, side, group index) owners of replayed groups
        (cached plans are shared across threads: the fill list is emptied
        only once every owner is in place)."""
        if not self._owner_fill:
            return
        with _OWNER_LOCK:
            owner = self._group_owner
            for g0, ei, owners in self._owner_fill:
                for j, (side, gi) in enumerate(owners):
                    owner[g0 + j] = (ei, side, gi)
            self._owner_fill = []

    def _group_slots(self, b: PlanBuilder, group_rows: list, chunks: list, s0: int, yop, zall: list,
                     n: int, owner_key: tuple) -> None:
        """Group slots of one replica group: chunk 0's tiles are those emitted
        since s0 (the compare / first replica segments); each further chunk
        gets a flat copy-0-vs-chunk segment of its own (when the copies are
        local) and its own slot."""
        first = len(group_rows)
        for j, (lo, hi) in enumerate(chunks):
            if j:
                s0 = b.tile_cursor
                if yop is not None:
                    b.add(None, 0, yop, 0, zall[lo - 1:hi - 1], 1, n, n, n)
            group_rows.append((s0, b.tile_cursor, hi - lo))
            self._group_owner.append(owner_key)
            self.group_offset.append(lo - 1)
        if len(chunks) > 1:
            self.subslots[first] = list(range(first, len(group_rows)))

    def slots_of(self, first_slot: int) -> list:
        """Every group slot of the replica group whose first slot is given."""
        return self.subslots.get(first_slot, [first_slot])

    def group_results(self, gres) -> dict:
        """{(entry, side): {group index: {"worst", "worst_index", "mismatch"}}}
        with a group's chunk slots folded the way check_replicas walks its
        copies (canonical.py:236-242): strict > over copies 1..m in order,
        so the first maximum wins and NaN never does."""
        out: dict = {}
        for row, key, off in zip(gres, self.group_owner, self.group_offset):
            ei, side, gi = key
            cur = out.setdefault((ei, side), {}).get(gi)
            w, wi, mm = float(row["worst"]), int(row["worst_index"]), int(row["mismatch"])
            if cur is None:
                out[(ei, side)][gi] = {"worst": w, "worst_index": wi + off if wi > 0 else wi, "mismatch": mm}
            else:
                if wi > 0 and w > cur["worst"]:
                    cur["worst"], cur["worst_index"] = w, wi + off
                cur["mismatch"] |= mm
        return out

    # tiles per SM worth aiming for before the default tile is shrunk
    TARGET_TILES = 148 * 8
    MIN_TILE_SHIFT = 8

    def _retile(self) -> int:
        """Shrink the tile below TD_TILE_UNITS when the plan is small.

        A tile is one CTA's unit of work; at the default 8192 units (128 KB
        per bf16 operand) a 1 MiB check has 8 tiles, so 8 SMs stream it
        through a chain of dependent DRAM round trips.  The largest
        2^k units (k >= 8, one unit per thread) that still yields about
        TARGET_TILES tiles is used instead, carried to the kernels in the
        segment flags.  Id / group tile ranges sit on segment boundaries, so
        they are remapped boundary to boundary.  Returns the shift stored in
        the flags (0 = the library default)."""
        b = self.builder
        cols = self._cols
        self.tile_units = N.TILE_UNITS
        default = N.TILE_UNITS.bit_length() - 1
        if not len(cols) or (1 << default) != N.TILE_UNITS:
            return 0
        units = cols[:, _C_NU]
        shift = default
        while shift > self.MIN_TILE_SHIFT and int((-(-units // (1 << shift))).sum()) < self.TARGET_TILES:
            shift -= 1
        if shift == default:
            return 0
        self.tile_units = 1 << shift
        counts = -(-units // self.tile_units)
        new_begin = np.concatenate([[0], np.cumsum(counts)])
        old_begin = np.append(cols[:, _C_TB], b.n_tiles)
        cols[:, _C_TB] = new_begin[:-1]
        b.n_tiles = self.n_tiles = int(new_begin[-1])

        def remap(v):
            return new_begin[np.searchsorted(old_begin, v)]
        for table in (self.ids, self.groups):
            if len(table):
                table["tile_begin"] = remap(table["tile_begin"])
                table["tile_end"] = remap(table["tile_end"])
        return shift

    # partial rows per chunk of the two-level slot reduction, and the largest
    # slot (in partial rows) below which one level is enough
    CHUNK_ROWS = 2048
    CHUNK_MIN_ROWS = int(os.environ.get("TD_CHUNK_MIN_ROWS", "8192"))

    def _chunk_slots(self) -> None:
        """Two-level slot reduction for plans with a big slot.

        td_finalize gives each id one CTA, which walks all of that id's
        partial rows: 8 per tile, so a 2 GB logits tensor is ~128 k rows on
        one SM.  When some slot exceeds CHUNK_MIN_ROWS rows, every slot's row
        range is cut into CHUNK_ROWS chunks (td_chunk table, reduced across
        the whole GPU by td_reduce_chunks), and `ids_chunked` /
        `groups_chunked` carry chunk ranges in place of tile ranges.  Sets
        self.chunks = None when one level suffices."""
        W = N.WARPS_PER_TILE
        rb = np.concatenate([self.ids["tile_begin"], self.groups["tile_begin"]]).astype(np.int64) * W
        re = np.concatenate([self.ids["tile_end"], self.groups["tile_end"]]).astype(np.int64) * W
        n_ids = len(self.ids)
        k0 = np.repeat(np.array([0, 2], np.int32), [n_ids, len(self.groups)])
        nk = np.concatenate([np.full(n_ids, 2, np.int32), 1 + self.groups["nz"].astype(np.int32)])
        self.chunks = None
        longest = int((re - rb).max()) if len(rb) else 0
        if longest < self.CHUNK_MIN_ROWS:
            return
        # chunks of CHUNK_ROWS for big slots; for mid-size plans (a few k rows,
        # e.g. a 4 MiB single-tensor check) chunks short enough that the
        # longest slot spreads over ~32 CTAs instead of one
        step = self.CHUNK_ROWS if longest >= 32 * self.CHUNK_ROWS else \
            min(self.CHUNK_ROWS, max(256, 1 << max(0, (longest // 32 - 1).bit_length())))
        # slot j -> chunks [c0[j], c1[j]) covering rows rb[j], rb[j]+step, ... < re[j]
        count = np.maximum(0, -(-(re - rb) // step))
        c1 = np.cumsum(count)
        c0 = c1 - count
        owner = np.repeat(np.arange(len(rb)), count)
        r0 = rb[owner] + (np.arange(int(c1[-1]) if len(c1) else 0, dtype=np.int64) - c0[owner]) * step
        chunks = np.zeros(len(r0), N.CHUNK)
        names = chunks.dtype.names
        chunks[names[0]], chunks[names[1]] = r0, np.minimum(r0 + step, re[owner])
        chunks[names[2]], chunks[names[3]] = k0[owner], nk[owner]
        self.chunks = chunks
        self.ids_chunked = self.ids.copy()
        self.ids_chunked["tile_begin"], self.ids_chunked["tile_end"] = c0[:n_ids], c1[:n_ids]
        self.groups_chunked = self.groups.copy()
        if len(self.groups):
            self.groups_chunked["tile_begin"] = c0[n_ids:]
            self.groups_chunked["tile_end"] = c1[n_ids:]

    # -- geometry -------------------------------------------------------------

    @staticmethod
    def _compare_runs(b: PlanBuilder, xmeta: IdMeta, y0, yop, zops, is_local) -> None:
        """Runs = candidate global boxes cut by reference global boxes."""
        for h in xmeta.groups:
            x0 = h.records[0]
            blocks = _run_blocks(y0.mapping, x0.mapping)
            if blocks:
                if not is_local(x0):
                    raise ValueError(
                        f"{x0.id.encode()}: the reference slice overlapping a candidate shard is not "
                        "on the rank holding that shard; give every rank the reference slices of "
                        "its candidate boxes")
                xop = b.operand(x0, x0.dtype_code)
                for xo, yo, rows, cols, rx, ry in blocks:
                    b.add(xop, xo, yop, yo, zops, rows, cols, rx, ry)

    def _settle_digest(self, b: PlanBuilder, first: int, y0, yop, remote_k: int, copy: int) -> None:
        """Keep the digest slot on a compare's segments only when they are all
        vector segments reading y0's payload and cover it exactly once (the
        reference boxes partition the candidate box); otherwise unstamp them
        (that copy is then digested by td_fingerprint)."""
        rows = b.seg_rows[first:]
        cells = sum(r[5] * r[6] for r in rows)
        ok = (rows and all(r[11] and r[2] is yop for r in rows)
              and cells == math.prod(y0.shape)
              and sum(loc.volume for loc, _ in y0.mapping.pairs) == math.prod(y0.shape))
        if ok:
            self.fused_digests.append((remote_k, copy))
        else:
            b.seg_rows[first:] = [r[:12] + (-1,) for r in rows]

    @staticmethod
    def _replica_remainder(b: PlanBuilder, y0, yop, zops) -> None:
        """Replica sums over payload cells no local box covers (usually none)."""
        shape = y0.mapping.local_shape
        covered = sum(loc.volume for loc, _ in y0.mapping.pairs)
        if covered == math.prod(shape):
            return
        pieces = [tuple((0, n) for n in shape)]
        for loc, _ in y0.mapping.pairs:
            nxt = []
            for p in pieces:
                nxt.extend(_subtract(p, loc.bounds))
            pieces = nxt
        for p in pieces:
            ext = tuple(hi - lo for lo, hi in p)
            st = tuple(lo for lo, _ in p)
            for _, yo, rows, cols, _, ry in _blocks(ext, st, shape, st, shape):
                b.add(None, 0, yop, yo, zops, rows, cols, ry, ry)

    # -- device tables ----------------------------------------------------------

    def _columns(self) -> None:
        """The segment rows as one int64 array (_TPL_NCOLS columns) in
        emission order: the general path's rows, and every replayed entry's
        template rows instantiated column-wise — per template, all of its
        replays at once, with their operand slots, first tile and digest slot
        offset — then merged back into emission order."""
        b = self.builder
        gen = np.array([(-1 if x is None else x.slot, xo, y.slot, yo,
                         *[z.slot for z in zs], *([-1] * (N.MAX_Z - len(zs))), len(zs),
                         r, c, rx, ry, tb, nu, int(vec), ds)
                        for x, xo, y, yo, zs, r, c, rx, ry, tb, nu, vec, ds in b.seg_rows],
                       np.int64).reshape(-1, _TPL_NCOLS)
        if not self._replays:
            self._cols = gen
            return
        rp = np.array(self._replays, np.int64)          # template, op0, tiles0, fd0
        pieces = [gen]
        order = np.argsort(rp[:, 0], kind="stable")
        cuts = np.flatnonzero(np.diff(rp[order, 0])) + 1
        for sel in np.split(order, cuts):
            rows = self._tpl_rows[int(rp[sel[0], 0])]
            m = len(rows)
            if m == 0:
                continue
            k = len(sel)
            R = np.repeat(rows[None, :, :], k, axis=0)
            S = R[:, :, _SLOT_COLS]
            R[:, :, _SLOT_COLS] = np.where(S >= 0, S + rp[sel, 1][:, None, None], S)
            R[:, :, _C_TB] += rp[sel, 2][:, None]
            D = R[:, :, _C_DS]
            R[:, :, _C_DS] = np.where(D >= 0, D + rp[sel, 3][:, None], D)
            pieces.append(R.reshape(k * m, _TPL_NCOLS))
        cols = np.concatenate(pieces)
        # every segment spans >= 1 tile and tiles are handed out in emission
        # order, so the first tile orders the segments as they were emitted
        self._cols = cols[np.argsort(cols[:, _C_TB], kind="stable")]

    def _freeze_segments(self) -> None:
        """The device segment table, tile -> segment map and per-class tile
        lists, built column-wise from _columns()' array."""
        cols = self._cols
        n = len(cols)
        segs = np.zeros(n, dtype=N.SEGMENT)
        self.operands = self.builder.operands
        self.operand_dtypes = self.builder.operand_dtypes
        if n == 0:
            self.seg_zslot = np.full((0, N.MAX_Z), -1, np.int64)
            self.seg_xslot = np.full(0, -1, np.int64)
            self.seg_xoff = self.seg_yslot = self.seg_yoff = np.zeros(0, np.int64)
            self.segs, self.tile_seg = segs, np.zeros(self.n_tiles, np.int32)
            self.class_keys, self.class_segs, self.class_lists = [], [], []
            self.algorithmic_bytes = 0
            return
        i64 = np.int64
        op_dt = np.asarray(self.operand_dtypes, np.int32)
        x_slot, y_slot = cols[:, _C_X].copy(), cols[:, _C_Y].copy()
        has_x = x_slot >= 0
        y_dt = op_dt[y_slot]
        y_es = _ESIZE[y_dt]
        x_dt = np.where(has_x, op_dt[np.maximum(x_slot, 0)], y_dt)
        x_es = np.where(has_x, _ESIZE[x_dt], 0)
        nz = cols[:, _C_NZ].astype(np.int32)
        self.seg_zslot = cols[:, _C_Z:_C_Z + N.MAX_Z].copy()
        r, c, rx, ry, tb, nu = (cols[:, k] for k in (_C_R, _C_C, _C_RX, _C_RY, _C_TB, _C_NU))
        xo, yo = cols[:, _C_XO], cols[:, _C_YO]
        vec = cols[:, _C_VEC] != 0
        ds = cols[:, _C_DS].astype(np.int32)
        segs["x_stride"], segs["y_stride"], segs["rows"], segs["cols"] = rx, ry, r, c
        segs["tile_begin"], segs["n_units"] = tb, nu
        segs["x_dtype"], segs["y_dtype"], segs["nz"] = x_dt, y_dt, nz
        segs["flags"] = ((has_x * N.SEG_HAS_X) | (vec * N.SEG_VEC)
                         | (self.tile_shift << N.SEG_TILE_SHIFT_POS)).astype(np.uint32)
        # _magic(d) for every row: p = 31 + bit_length(d - 1), m = ceil(2^p / d)
        d = np.where(vec, c // 8, c)
        _, e = np.frexp((d - 1).astype(np.float64))
        p = 31 + np.where(d > 1, e, 0).astype(i64)
        big = np.left_shift(np.ones(n, i64), p)
        m = big // d + (big % d != 0)
        segs["div_m"], segs["div_p"] = m.astype(np.uint32), p.astype(np.int32)
        segs["y_word0"], segs["digest_slot"] = (yo * y_es) // 8, ds
        self.seg_xslot, self.seg_xoff = x_slot, np.where(has_x, xo * x_es, 0)
        self.seg_yslot, self.seg_yoff = y_slot, yo * y_es
        nt = -(-nu // self.tile_units)
        seg_of_tile = np.repeat(np.arange(n, dtype=np.int32), nt)
        starts = np.concatenate([[0], np.cumsum(nt)[:-1]])
        if len(seg_of_tile) == self.n_tiles and np.array_equal(tb, starts):
            tile_seg = seg_of_tile                 # tiles handed out back to back (always, today)
        else:
            tile_seg = np.zeros(self.n_tiles, np.int32)
            tiles = np.repeat(tb - starts, nt) + np.arange(len(seg_of_tile), dtype=i64)
            tile_seg[tiles] = seg_of_tile
        # tile classes: (vector, y dtype, nz, has x, digest), sorted as tuples
        # packed one field per byte (every field < 256), so integer order is
        # the tuples' order
        code = ((((vec.astype(i64) << 8 | y_dt) << 8 | nz) << 8 | has_x) << 8) | (ds >= 0)
        uniq, inverse = np.unique(code, return_inverse=True)
        inverse = inverse.reshape(-1)
        self.segs = segs
        self.tile_seg = tile_seg
        self.class_keys = [(bool(k >> 32), int((k >> 24) & 255), int((k >> 16) & 255), bool((k >> 8) & 255),
                            bool(k & 255)) for k in uniq.tolist()]
        by_class = np.argsort(inverse, kind="stable")
        bounds = np.concatenate([[0], np.cumsum(np.bincount(inverse, minlength=len(uniq)))])
        self.class_segs = [by_class[bounds[k]:bounds[k + 1]].tolist() for k in range(len(uniq))]
        self.class_lists = []
        for k in range(len(uniq)):
            idx = by_class[bounds[k]:bounds[k + 1]].astype(i64)
            pick = np.repeat(idx, nt[idx])
            base = np.repeat(tb[idx] - np.concatenate([[0], np.cumsum(nt[idx])[:-1]]), nt[idx])
            t = base + np.arange(len(pick), dtype=i64)
            self.class_lists.append((pick << 32) + t)
        self.algorithmic_bytes = int((r * c * (y_es * (1 + nz) + x_es)).sum())

    # -- execution ----------------------------------------------------------------

    def run(self, pointers: np.ndarray, *, kappa: float = 3.0, eps: float = 0.0,
            replica_eps: float = 0.0, stream=None, timing: dict | None = None,
            sums: dict | None = None):
        """Execute once on the current CUDA device; pointers[k] is the device
        address of operand k.  Returns (id results, group results, near ties)."""
        prep = self.prepare(pointers, kappa=kappa, eps=eps, replica_eps=replica_eps, stream=stream)
        prep.launch(timing=timing)
        out = prep.fetch()
        if timing is not None:
            prep.read_timing(timing)
        if sums is not None:
            sums.update(prep.sums())
        return out

    def prepare(self, pointers: np.ndarray, *, kappa: float = 3.0, eps: float = 0.0,
                replica_eps: float = 0.0, stream=None, digests: int | None = None,
                tail_words: int = 0) -> "Prepared":
        """Patch live addresses into the segment table and stage every
        device-side table and workspace; the result can be launched repeatedly.
        digests: device address of the (len(fused_digests), 2) u64 table the
        digest classes accumulate into (the caller zeroes it per run).
        tail_words: f64 words reserved right after the slot sums, so that
        `exchange` = [slot sums | tail] is one contiguous buffer (the
        multi-GPU exchange buffer: sums, then digest rows)."""
        return Prepared(self, pointers, kappa, eps, replica_eps, stream, digests, tail_words)


_ONE_SEG = os.environ.get("TD_ONE_SEG", "1") != "0"      # A/B switch for by-value single segments
_STAGING_LOCK = threading.Lock()
_OWNER_LOCK = threading.Lock()


def _meta_key(meta):
    """Everything of an IdMeta the per-entry planner reads, as a hashable
    key: problems, hull, and per group its replica flags and every copy's
    (mapping signature id, dtype)."""
    if meta is None:
        return None
    if meta.struct_key is not None:
        return meta.struct_key
    return (meta.rank_problem, meta.merge_ok, meta.global_shape,
            tuple((g.numeric, g.declared_detail is None,
                   tuple((r.mapping.sig_id, r.dtype_code) for r in g.records)) for g in meta.groups))


_STRUCT_IDS: dict = {}
_STRUCT_COUNTER = itertools.count(1)


def _intern_struct(key: tuple) -> int:
    sid = _STRUCT_IDS.get(key)
    if sid is None:
        if len(_STRUCT_IDS) > (1 << 16):    # bound the table; ids stay unique (counter)
            _STRUCT_IDS.clear()
        sid = _STRUCT_IDS.setdefault(key, next(_STRUCT_COUNTER))
    return sid


def _owners_key(meta, owner):
    if meta is None:
        return None
    return tuple(tuple(owner(r) for r in g.records) for g in meta.groups)


def _shared_entries(entries) -> set:
    """Entries whose two sides hold the same record object (a trace checked
    against itself): operand de-duplication then differs from entry to entry,
    so they are planned without templates."""
    chain = itertools.chain.from_iterable
    xs = set(map(id, chain(e.x.all_records() for e in entries if e.x is not None)))
    if xs.isdisjoint(map(id, chain(e.y.all_records() for e in entries if e.y is not None))):
        return set()            # the usual case: two distinct traces
    return {ei for ei, e in enumerate(entries)
            if e.y is not None and any(id(r) in xs for g in e.y.groups for r in g.records)}


class Prepared:
    """A plan bound to payload addresses, with its tables resident in HBM."""

    def __init__(self, plan: Plan, pointers, kappa, eps, replica_eps, stream, digests=None, tail_words=0):
        import torch
        self.plan = plan
        self.kappa, self.eps, self.replica_eps = float(kappa), float(eps), float(replica_eps)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        n_ids, n_groups = len(plan.ids), len(plan.groups)
        self.n_ids, self.n_groups = n_ids, n_groups
        segs = plan.segs.copy()
        pointers = np.asarray(pointers, dtype=np.uint64)
        has_x = plan.seg_xslot >= 0
        segs["x"][has_x] = pointers[plan.seg_xslot[has_x]] + plan.seg_xoff[has_x].astype(np.uint64)
        segs["y"] = pointers[plan.seg_yslot] + plan.seg_yoff.astype(np.uint64)
        zmask = plan.seg_zslot >= 0
        zaddr = np.zeros(plan.seg_zslot.shape, dtype=np.uint64)
        zaddr[zmask] = pointers[plan.seg_zslot[zmask]] + \
            np.repeat(plan.seg_yoff[:, None], N.MAX_Z, 1)[zmask].astype(np.uint64)
        segs["z"] = zaddr
        # vector walkers need 16-byte aligned bases; operand resolution
        # (device.resolve_operands) guarantees it, so a violation is a bug
        if len(segs):
            vec = (segs["flags"] & N.SEG_VEC) != 0
            mis = ((segs["y"] % 16) != 0) | (has_x & ((segs["x"] % 16) != 0)) | \
                  (zmask & ((zaddr % 16) != 0)).any(axis=1)
            if (vec & mis).any():
                raise N.NativeError("vector segment with a misaligned operand address")
        dev = torch.device("cuda", torch.cuda.current_device())
        parts, offsets = [], []
        cursor = 0

        def put(arr):
            nonlocal cursor
            raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
            pad = (-cursor) % 16
            if pad:
                parts.append(np.zeros(pad, np.uint8))
                cursor += pad
            offsets.append(cursor)
            parts.append(raw)
            cursor += raw.size

        chunked = plan.chunks is not None
        groups = plan.groups_chunked if chunked else plan.groups
        gdesc = np.zeros(n_groups, N.GROUP_DESC)
        if n_groups:
            gdesc["tile_begin"] = groups["tile_begin"]
            gdesc["tile_end"] = groups["tile_end"]
            gdesc["nz"] = groups["nz"]
        put(segs)
        for lst in plan.class_lists:
            put(lst)
        put(plan.ids_chunked if chunked else plan.ids)
        put(gdesc)
        if chunked:
            put(plan.chunks)
        blob = np.concatenate(parts) if parts else np.zeros(16, np.uint8)
        # one pinned staging buffer per plan, reused by every binding of it
        # (cudaHostAlloc per check cost ~ms); the previous copy out of it must
        # have completed before it is overwritten
        # (a plan cached by check() can be bound by several threads at once:
        # the lock spans wait-for-previous-copy, fill and enqueue, so no
        # binding overwrites the buffer before another's copy has read it)
        self.tables = torch.empty(blob.size, dtype=torch.uint8, device=dev)
        with _STAGING_LOCK:
            staging, done = getattr(plan, "_staging", (None, None))
            if staging is None or staging.numel() < blob.size:
                staging = torch.empty(blob.size, dtype=torch.uint8).pin_memory()
            elif done is not None:
                done.synchronize()
            host = staging[:blob.size]
            host.numpy()[:] = blob
            with torch.cuda.stream(self.stream):
                self.tables.copy_(host, non_blocking=True)
                done = torch.cuda.Event()
                done.record(self.stream)
            plan._staging = (staging, done)
        self._host_blob = host                    # keep the pinned source alive
        base = self.tables.data_ptr()
        self.seg_ptr = base + offsets[0]
        n_cls = len(plan.class_lists)
        self.ids_ptr = base + offsets[1 + n_cls]
        self.grp_ptr = base + offsets[2 + n_cls]
        self.n_part = max(1, plan.n_tiles * N.WARPS_PER_TILE * N.PARTIAL_STRIDE)
        # ids / groups tables hold chunk ranges when the plan is chunked, and
        # the slot reduction then reads the chunk rows instead of the partials
        self.n_chunks = len(plan.chunks) if chunked else 0
        n_crow = self.n_chunks * N.WARPS_PER_TILE * N.PARTIAL_STRIDE
        self.n_slots = 2 * n_ids + N.SLOT_STRIDE * n_groups
        self.work = torch.empty(self.n_part + n_crow + self.n_slots + tail_words, dtype=torch.float64, device=dev)
        self.part_ptr = self.work.data_ptr()
        self.chunk_ptr = base + offsets[3 + n_cls] if chunked else 0
        self.red_ptr = self.part_ptr + 8 * self.n_part if chunked else self.part_ptr
        self.idsum_ptr = self.part_ptr + 8 * (self.n_part + n_crow)
        # the slot-sum vector (id sums, then group sums): what crosses ranks;
        # `exchange` extends it by the caller's tail (multi-GPU digests)
        self.exchange = self.work[self.n_part + n_crow:]
        self.slot_sums = self.exchange[:self.n_slots]
        self.gsum_ptr = self.idsum_ptr + 8 * 2 * n_ids
        self.res_bytes = N.ID_RESULT.itemsize * n_ids + N.GROUP_RESULT.itemsize * n_groups + 8
        self.res = torch.zeros(self.res_bytes, dtype=torch.uint8, device=dev)
        self.idres_ptr = self.res.data_ptr()
        self.gres_ptr = self.idres_ptr + N.ID_RESULT.itemsize * n_ids
        # the last 8 bytes: a u64 a caller may have a kernel write (the
        # multi-GPU digest-mismatch count), fetched with the results
        self.word_ptr = self.idres_ptr + self.res_bytes - 8
        self.last_word = 0
        # near ties are counted on the host from the per-id flags: no counter
        # reset between td_segnorm and the verdict kernel, which would keep
        # the verdict kernel from launching programmatically (PDL)
        self.tie_ptr = 0
        mode = N.MODE_STATIC if plan.static else N.MODE_NORMS
        atol, rtol = plan.static if plan.static else (0.0, 0.0)
        self.classes = np.zeros(len(plan.class_keys), N.CLASS)
        self.n_digests = len(plan.fused_digests)
        if self.n_digests and digests is None:
            self.digest_table = torch.zeros((self.n_digests, 2), dtype=torch.int64, device=dev)
            digests = self.digest_table.data_ptr()
        self.digest_ptr = digests or 0
        # single-segment classes hand their (patched) descriptor to the kernel
        # by value: host copies kept alive with this binding
        self._one_segs = []
        for k, (vec, dt, nz, hx, dg) in enumerate(plan.class_keys):
            host_seg = 0
            if len(plan.class_segs[k]) == 1 and vec and mode == N.MODE_NORMS and _ONE_SEG:
                one = segs[plan.class_segs[k][0]:plan.class_segs[k][0] + 1].copy()
                self._one_segs.append(one)
                host_seg = one.ctypes.data
            self.classes[k] = (base + offsets[1 + k], len(plan.class_lists[k]), dt, nz, int(hx),
                               int(vec), mode, int(dg), atol, rtol, self.digest_ptr if dg else 0, host_seg)
        self.launches_per_run = len(self.classes) + 1 + (1 if chunked else 0)
        self._events = None

    # -- the steps of one check (all stream-ordered, no host sync) ----------

    def segnorm(self, sh) -> None:
        if len(self.classes):
            N.call("td_segnorm", self.seg_ptr, self.classes.ctypes.data,
                   len(self.classes), self.part_ptr, 0, sh)

    def _chunks(self, sh) -> None:
        if self.n_chunks:
            N.call("td_reduce_chunks", self.part_ptr, self.chunk_ptr, self.n_chunks, self.red_ptr, sh)

    def reduce(self, sh) -> None:
        """partials -> per-slot sums (multi-GPU: all-reduced before verdict)."""
        self._chunks(sh)
        N.call("td_reduce_slots", self.ids_ptr, self.n_ids, self.grp_ptr, self.n_groups,
               self.red_ptr, self.idsum_ptr, self.gsum_ptr, sh)

    def verdict(self, sh) -> None:
        N.call("td_verdict", self.ids_ptr, self.n_ids, self.grp_ptr, self.n_groups,
               self.idsum_ptr, self.gsum_ptr, self.kappa, self.eps, self.replica_eps,
               self.idres_ptr, self.gres_ptr, self.tie_ptr, sh)

    def finalize(self, sh) -> None:
        """reduce + verdict, fused (single GPU)."""
        self._chunks(sh)
        N.call("td_finalize", self.ids_ptr, self.n_ids, self.grp_ptr, self.n_groups, self.red_ptr,
               self.idsum_ptr, self.gsum_ptr, self.kappa, self.eps, self.replica_eps,
               self.idres_ptr, self.gres_ptr, self.tie_ptr, sh)

    def launch(self, timing: dict | None = None) -> None:
        """Enqueue td_segnorm (one launch per tile class) and td_finalize
        (after td_reduce_chunks for a chunked plan) on the plan's stream; no
        host synchronisation."""
        import torch
        sh = N.stream_handle(self.stream)
        ev = None
        if timing is not None:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record(self.stream)
        self.segnorm(sh)
        if ev:
            ev[1].record(self.stream)
        self.finalize(sh)
        if ev:
            ev[2].record(self.stream)
        self._events = ev

    def capture(self):
        """A CUDA graph of launch(): replaying it re-runs the whole check
        (segnorm classes incl. their auxiliary-stream fork/join, finalize)
        with one host call — for checks small enough that launch latency
        dominates.  The graph reads whatever the bound payload buffers hold
        at replay time."""
        import torch
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(self.stream)
        keep, self.stream = self.stream, side
        try:
            with torch.cuda.graph(graph, stream=side):
                self.launch()
        finally:
            self.stream = keep
        self.stream.wait_stream(side)
        return graph

    def read_timing(self, timing: dict) -> None:
        ev = self._events
        if ev:
            ev[2].synchronize()
            timing["segnorm_ms"] = ev[0].elapsed_time(ev[1])
            timing["verdict_ms"] = ev[1].elapsed_time(ev[2])

    def fetch(self):
        """D2H of the packed results (synchronises the stream)."""
        import torch
        with torch.cuda.stream(self.stream):
            raw = self.res.cpu().numpy()
        n_ids, n_groups = self.n_ids, self.n_groups
        idres = raw[:N.ID_RESULT.itemsize * n_ids].view(N.ID_RESULT)
        lo = N.ID_RESULT.itemsize * n_ids
        gres = raw[lo:lo + N.GROUP_RESULT.itemsize * n_groups].view(N.GROUP_RESULT)
        ties = int(idres["near_tie"].sum()) if n_ids else 0
        self.last_word = int(raw[-8:].view(np.uint64)[0])
        return idres, gres, ties

    def sums(self) -> dict:
        """Per-id (d2, x2) and per-group (y2, z2...) sums, as reduced on the device."""
        with __import__("torch").cuda.stream(self.stream):
            flat = self.slot_sums.cpu().numpy()
        return {"id": flat[:2 * self.n_ids].reshape(self.n_ids, 2),
                "group": flat[2 * self.n_ids:].reshape(self.n_groups, N.SLOT_STRIDE)}


@functools.lru_cache(maxsize=65536)
def _run_blocks(ymap: ShardMapping, xmap: ShardMapping) -> tuple:
    """2-D blocks of (candidate pair x reference pair) box intersections
    (memoised on the two maps' signatures: every id of one layout shares them)."""
    key = (ymap.signature(), xmap.signature())
    out = _RUN_BLOCKS.get(key)
    if out is None:
        if len(_RUN_BLOCKS) > 65536:
            _RUN_BLOCKS.clear()
        out = _RUN_BLOCKS[key] = _run_blocks_uncached(ymap, xmap)
    return out


_RUN_BLOCKS: dict = {}


def _run_blocks_uncached(ymap: ShardMapping, xmap: ShardMapping) -> tuple:
    out = []
    for yl, yg in ymap.pairs:
        for xl, xg in xmap.pairs:
            cut = []
            for (a0, a1), (b0, b1) in zip(yg.bounds, xg.bounds):
                lo, hi = max(a0, b0), min(a1, b1)
                if lo >= hi:
                    cut = None
                    break
                cut.append((lo, hi))
            if cut is None:
                continue
            ext = tuple(hi - lo for lo, hi in cut)
            ys = tuple(l0 + (c0 - g0) for (l0, _), (g0, _), (c0, _) in zip(yl.bounds, yg.bounds, cut))
            xs = tuple(l0 + (c0 - g0) for (l0, _), (g0, _), (c0, _) in zip(xl.bounds, xg.bounds, cut))
            out.extend(_blocks(ext, xs, xmap.local_shape, ys, ymap.local_shape))
    return tuple(out)


def _replica_chunks(n_copies: int) -> list:
    """[(first copy, end copy)) ranges of at most MAX_Z replica copies (copy
    0 is every chunk's reference), at least one."""
    return [(lo, min(lo + N.MAX_Z, n_copies)) for lo in range(1, max(n_copies, 2), N.MAX_Z)]


def _group_dtype(records) -> int:
    """One dtype every copy of a replica group can be read as without loss."""
    codes = {r.dtype_code for r in records}
    if len(codes) == 1:
        return codes.pop()
    if N.F64 in codes:
        return N.F64
    return N.F32


def _subtract(box: tuple, cut: tuple) -> list:
    """box minus cut as disjoint boxes (bound tuples)."""
    inter = []
    for (a0, a1), (b0, b1) in zip(box, cut):
        lo, hi = max(a0, b0), min(a1, b1)
        if lo >= hi:
            return [box]
        inter.append((lo, hi))
    out = []
    rest = list(box)
    for axis, (lo, hi) in enumerate(inter):
        a0, a1 = rest[axis]
        if a0 < lo:
            piece = list(rest)
            piece[axis] = (a0, lo)
            out.append(tuple(piece))
        if hi < a1:
            piece = list(rest)
            piece[axis] = (hi, a1)
            out.append(tuple(piece))
        rest[axis] = (lo, hi)
    return out
