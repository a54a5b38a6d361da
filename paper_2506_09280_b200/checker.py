"""Trace comparison under perturbation-estimated tolerances — the drop-in
for pkg/src/traindiff/checker.py.

Same public surface and semantics: ToleranceMap (checker.py:49-99),
estimate_tolerance (:102-138), check (:312-365), CheckEntry / CheckReport /
render_report (:221-309, 446-489), compare_static (:403-443).  The
difference is where the arithmetic happens: metadata (grouping, hulls,
merge witnesses) is planned on the host by `plan`, and every norm, replica
check and threshold compare runs in the sm_100a kernels over payloads
resident in HBM.  `CheckPlan` exposes the plan so a layout that repeats
every step is planned once and re-run on fresh payloads.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _native as N
from .device import resolve_operands
from .errors import (ConfigInvalid, DigestMismatch, FormatError, ShapeMismatch,
                     TraindiffError)
from .perturb import PerturbSpec
from .plan import Plan, PlanEntry, gc_paused, merge_view, no_gc
from .tensor import FloatFormat
from .tracestore import Trace, canonical_json

VERDICT_PASS = "pass"
VERDICT_FLAG = "flag"
VERDICT_REPLICA = "replica-mismatch"
VERDICT_MERGE = "merge-error"
VERDICT_MISSING = "missing"
VERDICTS = (VERDICT_PASS, VERDICT_FLAG, VERDICT_REPLICA, VERDICT_MERGE, VERDICT_MISSING)
_NAME = {N.PASS: VERDICT_PASS, N.FLAG: VERDICT_FLAG, N.REPLICA: VERDICT_REPLICA,
         N.MERGE: VERDICT_MERGE}

Runner = Callable[[PerturbSpec | None], Trace]


@dataclass(frozen=True)
class ToleranceMap:
    """Per-id perturbation responses used as tolerances (checker.py:49-99)."""

    responses: dict
    n_samples: int
    eps_p: float
    aggregation: str = "max"

    def __post_init__(self):
        if self.n_samples < 1:
            raise ConfigInvalid("n_samples must be >= 1")
        if self.aggregation not in ("max", "mean"):
            raise ConfigInvalid(f"unknown aggregation {self.aggregation!r}")
        if not (self.eps_p >= 0.0 and math.isfinite(self.eps_p)):
            raise ConfigInvalid("eps_p must be finite and >= 0")
        for ident, resp in self.responses.items():
            if not (math.isfinite(resp) and resp >= 0.0):
                raise ConfigInvalid(f"response for {ident} must be finite and >= 0")

    def get(self, ident: str) -> float:
        """Never-estimated ids get 0.0, so the eps floor governs them."""
        return self.responses.get(ident, 0.0)

    def to_json(self) -> bytes:
        return canonical_json({"tolerance_version": 1, "n_samples": self.n_samples,
                               "eps_p": self.eps_p, "aggregation": self.aggregation,
                               "responses": self.responses})

    @classmethod
    def from_json(cls, blob) -> "ToleranceMap":
        try:
            doc = json.loads(blob)
        except (json.JSONDecodeError, UnicodeDecodeError) as exc:
            raise FormatError(f"tolerance file is not valid JSON: {exc}")
        if not isinstance(doc, dict) or doc.get("tolerance_version") != 1:
            raise FormatError("unsupported tolerance file version")
        try:
            return cls(responses={str(k): float(v) for k, v in doc["responses"].items()},
                       n_samples=int(doc["n_samples"]), eps_p=float(doc["eps_p"]),
                       aggregation=str(doc["aggregation"]))
        except (KeyError, TypeError, ValueError, AttributeError) as exc:
            raise FormatError(f"malformed tolerance file: {exc}")


@dataclass(frozen=True)
class CheckEntry:
    ident: str
    verdict: str
    observed: float | None
    tolerance: float | None
    threshold: float | None
    detail: str = ""


def _jsonable(value):
    if value is None:
        return None
    if not math.isfinite(value):
        return "inf" if value > 0 else ("-inf" if value < 0 else "nan")
    return value


def _entry_dicts(entries) -> list[dict]:
    return [{"id": e.ident, "verdict": e.verdict, "observed": _jsonable(e.observed),
             "tolerance": _jsonable(e.tolerance), "threshold": _jsonable(e.threshold),
             "detail": e.detail} for e in entries]


def _count(entries) -> dict[str, int]:
    counts = dict.fromkeys(VERDICTS, 0)
    for e in entries:
        counts[e.verdict] += 1
    return counts


def _first_with(entries, verdicts) -> str | None:
    return next((e.ident for e in entries if e.verdict in verdicts), None)


@dataclass(frozen=True)
class CheckReport:
    """Per-id outcomes in candidate execution order, reference-only ids last."""

    entries: tuple
    mode: str
    kappa: float
    fmt: FloatFormat
    near_ties: int = field(default=0, compare=False)

    @property
    def counts(self) -> dict[str, int]:
        return _count(self.entries)

    @property
    def earliest_flag(self) -> str | None:
        return _first_with(self.entries, (VERDICT_FLAG,))

    @property
    def earliest_divergence(self) -> str | None:
        return _first_with(self.entries, (VERDICT_FLAG, VERDICT_REPLICA, VERDICT_MERGE))

    def exit_code(self) -> int:
        """3 replica/merge failures, else 2 flags, else 0 (missing never gates)."""
        c = self.counts
        if c[VERDICT_REPLICA] or c[VERDICT_MERGE]:
            return 3
        return 2 if c[VERDICT_FLAG] else 0

    def to_dict(self) -> dict:
        return {"report_version": 1, "kind": "check", "mode": self.mode, "kappa": self.kappa,
                "format": self.fmt.value, "summary": self.counts,
                "earliest_flag": self.earliest_flag,
                "earliest_divergence": self.earliest_divergence,
                "exit_code": self.exit_code(), "entries": _entry_dicts(self.entries)}


def _require_same_setup(ref: Trace, cand: Trace) -> None:
    for key in ("digest", "mode"):
        a, b = ref.header.get(key), cand.header.get(key)
        if a != b:
            raise DigestMismatch(f"traces disagree on {key}: {a!r} vs {b!r}")


def _side_detail(meta, group_rows) -> str:
    """The first problem of one side in _merge_one's order: per group the
    declared-size or numeric replica problem, then the merge problem."""
    for gi, g in enumerate(meta.groups):
        if g.declared_detail is not None:
            return g.declared_detail
        row = group_rows.get(gi)
        if row is not None and row["mismatch"]:
            return (f"replicas diverge: rel_err {float(row['worst']):.6g} between ranks "
                    f"0 and {int(row['worst_index'])}")
    return meta.merge_detail or ""


class CheckPlan:
    """check() split into plan (metadata, once per layout) and run (GPU)."""

    @gc_paused
    def __init__(self, ref: Trace, cand: Trace, tol: ToleranceMap, kappa: float = 3.0, *,
                 fmt: FloatFormat):
        if kappa <= 0:
            raise ConfigInvalid("kappa must be positive")
        _require_same_setup(ref, cand)
        self.ref, self.cand, self.tol, self.kappa, self.fmt = ref, cand, tol, kappa, fmt
        self.ref_view = merge_view(ref)
        self.cand_view = merge_view(cand)
        self.common = [i for i in self.cand_view if i in self.ref_view]
        disjoint = set(map(id, ref.records)).isdisjoint(map(id, cand.records))
        self.plan = Plan([PlanEntry(i, x=self.ref_view[i], y=self.cand_view[i], x_rep=True,
                                    y_rep=True, tolerance=tol.get(i)) for i in self.common],
                         disjoint=disjoint)
        self.mode = str(cand.header.get("mode", ""))

    @property
    def algorithmic_bytes(self) -> int:
        return self.plan.algorithmic_bytes

    def execute(self, timing: dict | None = None, staged: dict | None = None, operands=None):
        """Device part only: resolve payloads, launch, fetch raw results.
        The host-side half of the report is built between the launch and the
        fetch, i.e. while host payloads are still crossing PCIe.  operands
        overrides the plan's payload owners (a cached plan bound to new
        traces of the same layout)."""
        ops = self.plan.operands if operands is None else operands
        ptrs, keep = resolve_operands(ops, self.plan.operand_dtypes, staged)
        prep = self.plan.prepare(ptrs, kappa=self.kappa, eps=self.fmt.eps, replica_eps=self.fmt.eps)
        prep.launch(timing=timing)
        self._report_rows()
        out = prep.fetch()
        if timing is not None:
            prep.read_timing(timing)
        del keep
        return out

    def run(self, timing: dict | None = None, staged: dict | None = None, operands=None) -> CheckReport:
        idres, gres, ties = self.execute(timing, staged, operands)
        return self.report(idres, gres, ties)

    def detach(self) -> list:
        """Drop every reference to the traces' payloads (for caching the plan
        across checks of one layout) and return, per plan operand, its
        (side, record position): 0 = reference, 1 = candidate."""
        pos = {id(r): (0, k) for k, r in enumerate(self.ref.records)}
        pos.update({id(r): (1, k) for k, r in enumerate(self.cand.records)})
        sources = [pos[id(o)] for o in self.plan.operands]
        for view in (self.ref_view, self.cand_view):
            for meta in view.values():
                meta.drop_records()
        self.plan.operands[:] = [None] * len(self.plan.operands)
        self.ref = self.cand = None
        return sources

    def _report_rows(self) -> list:
        """Everything of the report that does not depend on device results:
        per entry (ident, compare index or -1, tolerance, threshold, has
        compare, static detail), in report order (checker.py:328-365)."""
        rows = getattr(self, "_rows", None)
        if rows is not None:
            return rows
        kappa, eps = self.kappa, self.fmt.eps
        index = {ident: k for k, ident in enumerate(self.common)}
        has = self.plan.ids["has_compare"].tolist() if len(self.plan.ids) else []
        rows = []
        for ident, got in self.cand_view.items():
            tolerance = self.tol.get(ident)
            threshold = kappa * max(tolerance, eps)
            k = index.get(ident)
            if k is None:
                rows.append((ident, -1, tolerance, threshold, False, "only in candidate trace"))
                continue
            has_compare = bool(has[k])
            want = self.ref_view[ident]
            detail = "" if has_compare else (f"merged shapes differ: reference {want.global_shape} vs "
                                             f"candidate {got.global_shape}")
            rows.append((ident, k, tolerance, threshold, has_compare, detail))
        for ident in self.ref_view:
            if ident in self.cand_view:
                continue
            tolerance = self.tol.get(ident)
            rows.append((ident, -1, tolerance, kappa * max(tolerance, eps), False, "only in reference trace"))
        self._rows = rows
        return rows

    def report(self, idres, gres, ties) -> CheckReport:
        rows = self._report_rows()
        observed = idres["observed"].tolist()
        verdict = idres["verdict"].tolist()
        cand_kind = idres["cand_kind"].tolist()
        ref_kind = idres["ref_kind"].tolist()
        per_entry: dict | None = None
        entries = []
        for ident, k, tolerance, threshold, has_compare, detail in rows:
            if k < 0:
                entries.append(CheckEntry(ident, VERDICT_MISSING, None, tolerance, threshold, detail))
                continue
            if cand_kind[k] or ref_kind[k]:
                if per_entry is None:
                    per_entry = self.plan.group_results(gres)
                if cand_kind[k]:
                    detail = _side_detail(self.cand_view[ident], per_entry.get((k, 0), {}))
                else:
                    detail = "reference side: " + _side_detail(self.ref_view[ident], per_entry.get((k, 1), {}))
            entries.append(CheckEntry(ident, _NAME[verdict[k]], observed[k] if has_compare else None,
                                      tolerance, threshold, detail))
        return CheckReport(entries=tuple(entries), mode=self.mode, kappa=self.kappa, fmt=self.fmt,
                           near_ties=ties)


def check(ref: Trace, cand: Trace, tol: ToleranceMap, kappa: float = 3.0, *,
          fmt: FloatFormat) -> CheckReport:
    """Compare a candidate trace against the reference (checker.py:312-365):
    replica copies must agree to fmt precision, shards are merged (never
    materialised here), and an id flags when rel_err(ref, cand) exceeds
    kappa * max(tolerance, fmt.eps).

    Host-resident payloads start their H2D copies before planning, so the
    metadata work overlaps the DMA.  Host traces larger than the device's
    free memory are checked in consecutive batches of ids (the reference
    checks host traces of any size), with the same report."""
    if kappa <= 0:
        raise ConfigInvalid("kappa must be positive")
    _require_same_setup(ref, cand)
    host = _host_bytes(ref) + _host_bytes(cand)
    if host:                          # device-resident traces skip the free-memory query
        budget = _hbm_budget(host)
        if budget is not None and host > budget:
            return _check_in_batches(ref, cand, tol, kappa, fmt, budget)
    return _check_direct(ref, cand, tol, kappa, fmt, resident=not host)


def _check_direct(ref: Trace, cand: Trace, tol: ToleranceMap, kappa: float, fmt: FloatFormat,
                  resident: bool = False) -> CheckReport:
    """check() with every payload staged on the device at once (resident:
    every payload is already in device memory, nothing to stage)."""
    from .device import stage_host_payloads
    staged = {} if resident else stage_host_payloads([ref, cand])
    key = _check_key(ref, cand, tol, kappa, fmt)
    hit = _PLAN_CACHE.get(key)
    if hit is not None:
        # same layout as a previous check: reuse its plan (metadata only) and
        # bind this check's payloads by record position
        cp, sources = hit
        traces = (ref.records, cand.records)
        return cp.run(staged=staged, operands=[traces[side][k] for side, k in sources])
    cp = CheckPlan(ref, cand, tol, kappa, fmt=fmt)
    report = cp.run(staged=staged)
    if len(_PLAN_CACHE) >= _PLAN_CACHE_SIZE:
        _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
    _PLAN_CACHE[key] = (cp, cp.detach())
    return report


def _host_bytes(trace: Trace) -> int:
    """Payload bytes check() would have to bring to the device."""
    ext = N.host_ext()
    if ext is not None:
        total = ext.host_bytes(trace.records)
        if total is not None:
            return total
    return _host_bytes_py(trace)


def _host_bytes_py(trace: Trace) -> int:
    total = 0
    for r in trace.records:
        p = r.payload
        if not (getattr(p, "is_cuda", False)):
            total += r.nbytes
    return total


def _hbm_budget(host_bytes: int = 0) -> int | None:
    """Device bytes a check may stage at once: TD_HBM_BUDGET_BYTES, else the
    free HBM less a margin for plan tables and workspace (None without a
    GPU: check() then fails loudly further down, as before).  The driver's
    free-memory query costs 10-20 ms per call on a loaded device, so it is
    made only when the host bytes could come near the limit: below half of
    what this process has not allocated, the answer cannot be 'batch'."""
    import os
    env = os.environ.get("TD_HBM_BUDGET_BYTES")
    if env:
        return int(env)
    try:
        import torch
        if not torch.cuda.is_available():
            return None
        dev = torch.cuda.current_device()
        headroom = torch.cuda.get_device_properties(dev).total_memory - torch.cuda.memory_allocated(dev)
        if 2 * host_bytes + (4 << 30) < headroom:
            return headroom
        free, _ = torch.cuda.mem_get_info()
        free += torch.cuda.memory_reserved() - torch.cuda.memory_allocated()   # the allocator's cache
    except Exception:  # pragma: no cover - no driver
        return None
    return int(free * 0.9) - (1 << 30)


def _check_in_batches(ref: Trace, cand: Trace, tol: ToleranceMap, kappa: float, fmt: FloatFormat,
                      budget: int) -> CheckReport:
    """check() of host traces larger than the device: the candidate's ids,
    in execution order, are cut into consecutive batches whose payloads (both
    sides) fit `budget`; each batch is an ordinary check of the two traces
    restricted to its ids (every id's verdict depends on its own records
    only), and the entries are concatenated in the same order — candidate
    execution order, then reference-only ids — so the report is the one
    check() of the whole traces gives (checker.py:328-365)."""
    cand_ids = cand.by_id()
    ref_ids = ref.by_id()
    size = {}
    for trace in (ref, cand):
        for r in trace.records:
            if not getattr(r.payload, "is_cuda", False):
                ident = r.id.encode()
                size[ident] = size.get(ident, 0) + r.nbytes
    batches, cur, used = [], [], 0
    for ident in cand_ids:
        nb = size.get(ident, 0)
        if cur and used + nb > budget:
            batches.append(cur)
            cur, used = [], 0
        cur.append(ident)
        used += nb
    if cur:
        batches.append(cur)
    entries, ties = [], 0
    for ids in batches:
        keep = set(ids)
        sub_ref = Trace(header=ref.header, raw_header=ref.raw_header,
                        records=[r for r in ref.records if r.id.encode() in keep])
        sub_cand = Trace(header=cand.header, raw_header=cand.raw_header,
                         records=[r for r in cand.records if r.id.encode() in keep])
        rep = _check_direct(sub_ref, sub_cand, tol, kappa, fmt)
        entries.extend(rep.entries)
        ties += rep.near_ties
    eps = fmt.eps
    for ident in ref_ids:
        if ident not in cand_ids:
            tolerance = tol.get(ident)
            entries.append(CheckEntry(ident, VERDICT_MISSING, None, tolerance, kappa * max(tolerance, eps),
                                      "only in reference trace"))
    return CheckReport(entries=tuple(entries), mode=str(cand.header.get("mode", "")), kappa=kappa, fmt=fmt,
                       near_ties=ties)


# check() plans are pure functions of the traces' metadata, the tolerances,
# kappa and the format: the last few are kept (payload references dropped),
# so repeated checks of one layout — every step of a run, every sample of a
# sweep — skip the host planner (~0.1 s for config 2).
_PLAN_CACHE: dict = {}
_PLAN_CACHE_SIZE = 4


def _check_key(ref: Trace, cand: Trace, tol: ToleranceMap, kappa: float, fmt: FloatFormat) -> tuple:
    return (_layout_key(ref), _layout_key(cand), ref.header.get("mode"), cand.header.get("mode"),
            frozenset(tol.responses.items()), float(kappa), fmt)


def _strict_problem(view, plan: Plan, gres, side_of_entry: dict) -> str | None:
    """First id (view order) with a merge/replica problem, as 'id: detail'."""
    per_entry = plan.group_results(gres)
    for ident, meta in view.items():
        rows = per_entry.get(side_of_entry[ident], {})
        numeric = any(r["mismatch"] for r in rows.values())
        if meta.declared_problem is not None or numeric or not meta.merge_ok:
            return f"{ident}: {_side_detail(meta, rows)}"
    return None


def _layout_key(trace) -> tuple:
    """Everything a plan depends on, per record, in trace order: ids, rank
    metas, mapping signatures (as their interned ids: equal ids = equal
    signatures), dtypes, payload shapes, replica sizes — column by column
    (no tuple per record) and with the cyclic GC paused: every check() of a
    cached layout builds and compares this key before it launches anything."""
    ext = N.host_ext()
    if ext is not None:
        return ext.layout_key(trace.records)
    return _layout_key_py(trace)


def _layout_key_py(trace) -> tuple:
    recs = trace.records
    with no_gc():
        return (tuple([r.id.encode() for r in recs]), tuple([r.rank_meta.as_tuple() for r in recs]),
                tuple([r.mapping.sig_id for r in recs]), tuple([r.dtype_code for r in recs]),
                tuple([r.payload.shape for r in recs]), tuple([r.replica_group_size for r in recs]))


def _forget_payloads(view, plan: Plan, keep_ids) -> None:
    """Drop a sample trace's record references from a cached view / plan
    (the cached path re-binds operands by position and reads only metadata)."""
    for meta in view.values():
        meta.drop_records()
    plan.operands[:] = [o if id(o) in keep_ids else None for o in plan.operands]


def estimate_tolerance(runner: Runner, *, n_samples: int = 5, eps_p: float,
                       aggregation: str = "max") -> ToleranceMap:
    """Per-id response to an eps_p input nudge (checker.py:102-138).

    runner(None) replays the trusted run; runner(PerturbSpec(s, eps_p))
    replays it perturbed (the B200 runner applies td_perturb in a hook).
    Merges are strict with FP32 replica tolerance, as in the reference."""
    if n_samples < 1:
        raise ConfigInvalid("n_samples must be >= 1")
    if aggregation not in ("max", "mean"):
        raise ConfigInvalid(f"unknown aggregation {aggregation!r}")
    rep_eps = FloatFormat.FP32.eps
    base_trace = runner(None)
    base = merge_view(base_trace)
    plan = Plan([PlanEntry(i, x=None, y=m, x_rep=False, y_rep=True) for i, m in base.items()])
    ptrs, keep = resolve_operands(plan.operands, plan.operand_dtypes)
    _, gres, _ = plan.run(ptrs, replica_eps=rep_eps)
    del keep
    problem = _strict_problem(base, plan, gres, {i: (k, 0) for k, i in enumerate(base)})
    if problem is not None:
        raise TraindiffError(problem)
    samples: dict = {ident: [] for ident in base}
    base_pos = {id(r): k for k, r in enumerate(base_trace.records)}
    cached = None          # (layout key, plan, view, operand sources)
    for s in range(n_samples):
        trace = runner(PerturbSpec(sample=s, eps=eps_p))
        key = _layout_key(trace)
        if cached is not None and cached[0] == key:
            # same layout as the previous sample: reuse the plan and bind the
            # new payloads by record position (metadata is data-independent)
            _, plan, pert, sources = cached
            owners = [base_trace.records[k] if from_base else trace.records[k]
                      for from_base, k in sources]
            ptrs, keep = resolve_operands(owners, plan.operand_dtypes)
        else:
            pert = merge_view(trace)
            plan = Plan([PlanEntry(ident, x=base.get(ident), y=meta, x_rep=False, y_rep=True)
                         for ident, meta in pert.items()])
            pos = {id(r): k for k, r in enumerate(trace.records)}
            sources = [(True, base_pos[id(o)]) if id(o) in base_pos else (False, pos[id(o)])
                       for o in plan.operands]
            cached = (key, plan, pert, sources)
            ptrs, keep = resolve_operands(plan.operands, plan.operand_dtypes)
        idres, gres, _ = plan.run(ptrs, replica_eps=rep_eps)
        del keep
        problem = _strict_problem(pert, plan, gres, {i: (k, 0) for k, i in enumerate(pert)})
        if problem is not None:
            raise TraindiffError(problem)
        index = {ident: k for k, ident in enumerate(pert)}
        for ident, meta in base.items():
            k = index.get(ident)
            if k is None:
                continue
            moved = pert[ident]
            if meta.global_shape != moved.global_shape:
                raise ShapeMismatch(f"rel_err: {meta.global_shape} vs {moved.global_shape}")
            resp = float(idres[k]["observed"])
            samples[ident].append(resp if math.isfinite(resp) else 0.0)
        # hold no payload of this sample while the next one runs: only one
        # perturbed trace is alive at a time (with the base), so a run whose
        # traces are a third of HBM still fits
        _forget_payloads(pert, plan, base_pos)
        del trace, ptrs
    responses = {}
    for ident, resp in samples.items():
        if not resp:
            responses[ident] = 0.0
        elif aggregation == "max":
            responses[ident] = max(resp)
        else:
            responses[ident] = sum(resp) / len(resp)
    return ToleranceMap(responses=responses, n_samples=n_samples, eps_p=eps_p,
                        aggregation=aggregation)


def estimate_tolerance_streaming(runner, *, n_samples: int = 5, eps_p: float,
                                 aggregation: str = "max") -> ToleranceMap:
    """estimate_tolerance (checker.py:102-138) without materialising the
    perturbed traces: a B200 extension for single-GPU traced runs.

    runner(None) returns the base Trace (device-resident, one identity-mapped
    record per id, e.g. runner.torch_runner); runner(spec, sink=f) replays
    the perturbed step and hands every capture to f instead of keeping it.
    Each capture is compared with its base record the moment it is produced
    — td_rel_err enqueued on the capturing stream, its sums written to a
    per-(sample, id) slot in HBM, no host sync — so the compare overlaps the
    model's own compute and only the base trace stays resident (config 4 at
    S=8192: ~75 GB of traces instead of ~150).  Same semantics as
    estimate_tolerance: rel_err(base, perturbed) per id, non-finite -> 0.0,
    ids absent from a sample skipped, max / mean aggregation."""
    import torch
    from .device import pair_sums
    if n_samples < 1:
        raise ConfigInvalid("n_samples must be >= 1")
    if aggregation not in ("max", "mean"):
        raise ConfigInvalid(f"unknown aggregation {aggregation!r}")
    base = {ident: x for ident, (_, x) in _identity_records(runner(None), "streaming estimation").items()}
    ids = list(base)
    index = {ident: k for k, ident in enumerate(ids)}
    sums = torch.zeros((n_samples, max(len(ids), 1), 3), dtype=torch.float64, device="cuda")
    work = torch.zeros(N.REL_ERR_WORK_BYTES, dtype=torch.uint8, device="cuda")
    present = []
    for s in range(n_samples):
        got: dict = {}

        def sink(ident, tensor, module_class, _s=s, _got=got):
            x = base.get(ident)
            if x is None:
                return                                  # not in the base trace: ignored
            y = tensor.reshape(-1)
            if y.numel() != x.numel():
                raise ShapeMismatch(f"rel_err: {ident} has {y.numel()} elements vs {x.numel()}")
            k = index[ident]
            if y.dtype == x.dtype:
                N.call("td_rel_err", x.data_ptr(), y.data_ptr(), N.dtype_code(x), x.numel(),
                       work.data_ptr(), sums[_s, k].data_ptr(), N.stream_handle())
                _got[ident] = None
            else:                                       # mixed dtypes: widening path, synchronous
                _got[ident] = pair_sums(x.double(), y.double())[2]
        runner(PerturbSpec(sample=s, eps=eps_p), sink=sink)
        present.append(got)
    rel = sums[:, :, 2].cpu().numpy()
    responses = {}
    for ident in ids:
        k = index[ident]
        resp = []
        for s in range(n_samples):
            if ident not in present[s]:
                continue
            v = present[s][ident]
            v = float(rel[s, k]) if v is None else v
            resp.append(v if math.isfinite(v) else 0.0)
        if not resp:
            responses[ident] = 0.0
        elif aggregation == "max":
            responses[ident] = max(resp)
        else:
            responses[ident] = sum(resp) / len(resp)
    return ToleranceMap(responses=responses, n_samples=n_samples, eps_p=eps_p, aggregation=aggregation)


def _identity_records(trace: Trace, what: str) -> dict:
    """{id: (record, flat device payload)} of a single-GPU trace (one
    identity-mapped record per id) — what the streaming entry points need."""
    from .canonical import identity_mapping
    from .device import to_device
    out: dict = {}
    for rec in trace.records:
        ident = rec.id.encode()
        if ident in out:
            raise ConfigInvalid(f"{ident}: {what} needs one record per id (single GPU)")
        if rec.replica_group_size != 1 or \
                rec.mapping.signature() != identity_mapping(tuple(rec.mapping.global_shape)).signature():
            raise ConfigInvalid(f"{ident}: {what} needs identity-mapped records")
        out[ident] = (rec, to_device(rec.payload).reshape(-1))
    return out


def check_streaming(ref: Trace, run: Callable, tol: ToleranceMap, kappa: float = 3.0, *,
                    fmt: FloatFormat) -> CheckReport:
    """check() (checker.py:312-365) of a LIVE candidate step against a
    resident single-GPU reference trace, without materialising the candidate
    trace: a B200 extension.

    run(sink) executes the candidate's traced step, handing every capture to
    sink(ident, tensor, module_class) — e.g. `lambda sink: runner(None,
    sink=sink)` with runner.torch_runner.  Each capture is compared with its
    reference record as it is produced (td_rel_err on the capturing stream,
    sums to a per-id HBM slot, no host sync).  The report is check()'s:
    candidate execution order, then reference-only ids; threshold kappa *
    max(tol, fmt.eps); NaN passes, +inf flags; differing shapes are merge
    errors; ids on one side only are missing."""
    import torch
    from .device import pair_sums
    if kappa <= 0:
        raise ConfigInvalid("kappa must be positive")
    base = _identity_records(ref, "check_streaming")
    index = {ident: k for k, ident in enumerate(base)}
    sums = torch.zeros((max(len(base), 1), 3), dtype=torch.float64, device="cuda")
    work = torch.zeros(N.REL_ERR_WORK_BYTES, dtype=torch.uint8, device="cuda")
    order: list = []
    shapes: dict = {}

    def sink(ident, tensor, module_class):
        order.append(ident)
        entry = base.get(ident)
        if entry is None:
            return
        rec, x = entry
        if tuple(tensor.shape) != tuple(rec.mapping.global_shape):
            shapes[ident] = tuple(tensor.shape)
            return
        y = tensor.reshape(-1)
        if y.dtype == x.dtype:
            N.call("td_rel_err", x.data_ptr(), y.data_ptr(), N.dtype_code(x), x.numel(),
                   work.data_ptr(), sums[index[ident]].data_ptr(), N.stream_handle())
        else:                                           # mixed dtypes: widening path, synchronous
            d2, a2, _ = pair_sums(x.double(), y.double())
            sums[index[ident], 0], sums[index[ident], 1] = d2, a2
    run(sink)
    # verdicts in the batched verdict kernel, as check()'s (td_verdict:
    # precedence, threshold kappa * max(tol, eps), NaN passes, near ties)
    eps = fmt.eps
    n = len(base)
    desc = np.zeros(max(n, 1), dtype=N.ID_DESC)
    seen = set(order)
    for ident, k in index.items():
        desc[k]["tolerance"] = tol.get(ident)
        desc[k]["has_compare"] = int(ident in seen and ident not in shapes)
        desc[k]["cand_host"] = N.MERGE if ident in shapes else 0
    res = np.zeros(max(n, 1), dtype=N.ID_RESULT)
    if n:
        dev_desc = torch.from_numpy(desc.view(np.uint8)).to("cuda")
        id_sums = sums[:, :2].contiguous()
        dev_res = torch.zeros(res.nbytes, dtype=torch.uint8, device="cuda")
        dev_ties = torch.zeros(1, dtype=torch.int64, device="cuda")
        N.call("td_verdict", dev_desc.data_ptr(), n, 0, 0, id_sums.data_ptr(), 0, float(kappa), float(eps),
               float(eps), dev_res.data_ptr(), 0, dev_ties.data_ptr(), N.stream_handle())
        res = dev_res.cpu().numpy().view(N.ID_RESULT)
    entries, ties = [], 0
    for ident in order:
        tolerance = tol.get(ident)
        threshold = kappa * max(tolerance, eps)
        entry = base.get(ident)
        if entry is None:
            entries.append(CheckEntry(ident, VERDICT_MISSING, None, tolerance, threshold,
                                      "only in candidate trace"))
            continue
        row = res[index[ident]]
        if ident in shapes:
            entries.append(CheckEntry(ident, _NAME[int(row["verdict"])], None, tolerance, float(row["threshold"]),
                                      f"merged shapes differ: reference {tuple(entry[0].mapping.global_shape)} "
                                      f"vs candidate {shapes[ident]}"))
        else:
            ties += int(row["near_tie"])
            entries.append(CheckEntry(ident, _NAME[int(row["verdict"])], float(row["observed"]), tolerance,
                                      float(row["threshold"]), ""))
    for ident in base:
        if ident not in seen:
            tolerance = tol.get(ident)
            entries.append(CheckEntry(ident, VERDICT_MISSING, None, tolerance, kappa * max(tolerance, eps),
                                      "only in reference trace"))
    return CheckReport(entries=tuple(entries), mode=str(ref.header.get("mode", "")), kappa=kappa, fmt=fmt,
                       near_ties=int(ties))


# ---------------------------------------------------------------------------
# static-threshold ablation and rendering

@dataclass(frozen=True)
class StaticReport:
    """Fixed-threshold baseline outcome (checker.py:368-400)."""

    entries: tuple
    atol: float
    rtol: float

    @property
    def counts(self) -> dict[str, int]:
        return _count(self.entries)

    @property
    def earliest_flag(self) -> str | None:
        return _first_with(self.entries, (VERDICT_FLAG,))

    def exit_code(self) -> int:
        c = self.counts
        if c[VERDICT_MERGE]:
            return 3
        return 2 if c[VERDICT_FLAG] else 0

    def to_dict(self) -> dict:
        return {"report_version": 1, "kind": "static", "atol": self.atol, "rtol": self.rtol,
                "summary": self.counts, "earliest_flag": self.earliest_flag,
                "exit_code": self.exit_code(), "entries": _entry_dicts(self.entries)}


def compare_static(ref: Trace, cand: Trace, atol: float, rtol: float) -> StaticReport:
    """Elementwise |cand - ref| <= atol + rtol*|ref| per id, no replica
    checks (checker.py:403-443); the elementwise test runs in td_segnorm's
    static mode."""
    if atol < 0 or rtol < 0:
        raise ConfigInvalid("atol and rtol must be nonnegative")
    _require_same_setup(ref, cand)
    ref_view = merge_view(ref, replica_check=False)
    cand_view = merge_view(cand, replica_check=False)
    common = [i for i in cand_view if i in ref_view]
    plan = Plan([PlanEntry(i, x=ref_view[i], y=cand_view[i], x_rep=False, y_rep=False)
                 for i in common], static=(float(atol), float(rtol)))
    ptrs, keep = resolve_operands(plan.operands, plan.operand_dtypes)
    sums: dict = {}
    plan.run(ptrs, sums=sums)
    del keep
    index = {ident: k for k, ident in enumerate(common)}
    entries = []
    for ident, got in cand_view.items():
        k = index.get(ident)
        if k is None:
            entries.append(CheckEntry(ident, VERDICT_MISSING, None, None, None,
                                      "only in candidate trace"))
            continue
        want = ref_view[ident]
        if not got.merge_ok:
            entries.append(CheckEntry(ident, VERDICT_MERGE, None, None, None, got.merge_detail))
        elif not want.merge_ok:
            entries.append(CheckEntry(ident, VERDICT_MERGE, None, None, None,
                                      f"reference side: {want.merge_detail}"))
        elif want.global_shape != got.global_shape:
            entries.append(CheckEntry(ident, VERDICT_MERGE, None, None, None,
                                      f"merged shapes differ: reference {want.global_shape} vs "
                                      f"candidate {got.global_shape}"))
        else:
            failing = sums["id"][k, 0]
            entries.append(CheckEntry(ident, VERDICT_PASS if failing == 0 else VERDICT_FLAG,
                                      None, None, None))
    for ident in ref_view:
        if ident not in cand_view:
            entries.append(CheckEntry(ident, VERDICT_MISSING, None, None, None,
                                      "only in reference trace"))
    return StaticReport(entries=tuple(entries), atol=atol, rtol=rtol)


def _fmt_value(value) -> str:
    return "-" if value is None else f"{value:.6g}"


def _render_text(report) -> str:
    doc = report.to_dict()
    if doc["kind"] == "check":
        lines = [f"check mode={doc['mode']} kappa={doc['kappa']:g} format={doc['format']}"]
    else:
        lines = [f"static check atol={doc['atol']:g} rtol={doc['rtol']:g}"]
    earliest = doc["earliest_flag"]
    for e in report.entries:
        mark = ">" if earliest is not None and e.ident == earliest else " "
        line = (f"{mark} {e.verdict:<16} obs={_fmt_value(e.observed):>12} "
                f"tol={_fmt_value(e.tolerance):>12} thr={_fmt_value(e.threshold):>12}  {e.ident}")
        if e.detail:
            line += f"  [{e.detail}]"
        lines.append(line)
    counts = report.counts
    lines.append("summary: " + ", ".join(f"{counts[v]} {v}" for v in VERDICTS))
    lines.append(f"earliest flag: {earliest if earliest else '(none)'}")
    divergence = doc.get("earliest_divergence")
    if divergence is not None and divergence != earliest:
        lines.append(f"earliest divergence: {divergence}")
    return "\n".join(lines) + "\n"


def render_report(report, format: str = "text") -> str:
    if format == "json":
        return canonical_json(report.to_dict()).decode("utf-8")
    if format == "text":
        return _render_text(report)
    raise ConfigInvalid(f"unknown report format {format!r}")
