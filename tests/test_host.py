"""CPU-only tests of the host side: data-free merge witnesses, the TTRC
codec, report rendering and plan metadata, checked against the golden
fixtures the reference produced and against the oracle."""

import json
import math

import numpy as np
import pytest

from oracle import traindiff_oracle as O
from paper_2506_09280_b200 import canonical as C
from paper_2506_09280_b200.canonical import ShardMapping, SliceBox
from paper_2506_09280_b200.checker import (CheckEntry, CheckReport, ToleranceMap,
                                           render_report)
from paper_2506_09280_b200.errors import ConfigInvalid, FormatError, MergeConflict
from paper_2506_09280_b200.plan import merge_view
from paper_2506_09280_b200.tensor import FloatFormat
from paper_2506_09280_b200.tracestore import trace_from_bytes, trace_to_bytes


def _mapping(sig):
    pairs = tuple((SliceBox(tuple(map(tuple, l))), SliceBox(tuple(map(tuple, g))))
                  for l, g in sig["pairs"])
    return ShardMapping(tuple(sig["local_shape"]), tuple(sig["global_shape"]), pairs)


def test_data_free_witnesses_match_reference(shardings):
    """The boxes-only overlap/gap witnesses equal the reference merge's
    count-array witnesses on the 1000 randomized shardings (x3 variants)."""
    for case in shardings:
        shape = tuple(case["shape"])
        maps = [_mapping(s) for s in case["shards"]]
        v = case["victim"]
        for key, ms in (("ok", maps), ("omitted", maps[:v] + maps[v + 1:]),
                        ("doubled", maps + [maps[v]])):
            err = C.merge_problem(ms, shape)
            want = case[key]
            if want is None:
                assert err is None
            else:
                assert isinstance(err, MergeConflict)
                assert str(err) == want["message"]
                assert list(err.witness) == want["witness"]


def test_mapping_problem_matches_count_array_oracle():
    rng = np.random.default_rng(3)
    for _ in range(2000):
        nd = int(rng.integers(0, 4))
        local = tuple(int(rng.integers(0, 5)) for _ in range(nd))
        pairs = []
        for _ in range(int(rng.integers(0, 4))):
            lb = []
            gb = []
            for n in local:
                a = int(rng.integers(0, n + 2))
                b = a + int(rng.integers(0, 3))
                lb.append((a, b))
                g0 = int(rng.integers(0, 3))
                gb.append((g0, g0 + (b - a) + (1 if rng.random() < 0.1 else 0)))
            pairs.append((tuple(lb), tuple(gb)))
        glob = tuple(n + 2 for n in local)
        want = O.validate_mapping(local, glob, pairs)
        m = ShardMapping(local, glob, tuple((SliceBox(l), SliceBox(g)) for l, g in pairs))
        assert C.mapping_problem(m) == want


def test_ttrc_round_trip_is_byte_identical(cases, golden_trace_bytes):
    for name in cases["traces"]:
        raw = golden_trace_bytes(name)
        trace = trace_from_bytes(raw)
        assert trace_to_bytes(trace) == raw, name


@pytest.mark.parametrize("bad,offset", [(b"XXXX", 0)])
def test_ttrc_rejects_bad_magic(bad, offset, golden_trace_bytes):
    raw = bad + golden_trace_bytes("fp32_ref_m1")[4:]
    with pytest.raises(FormatError) as info:
        trace_from_bytes(raw)
    assert info.value.offset == offset


def test_ttrc_truncation_is_a_format_error(golden_trace_bytes):
    raw = golden_trace_bytes("fp32_ref_m1")
    for cut in range(0, len(raw) - 1, max(1, len(raw) // 97)):
        with pytest.raises(FormatError):
            trace_from_bytes(raw[:cut])


def test_render_matches_reference_text(cases):
    """Our renderer reproduces the reference's text and JSON reports byte for
    byte when fed the reference's own entries."""
    for case in cases["checks"]:
        doc = json.loads(case["report"])
        entries = tuple(CheckEntry(e["id"], e["verdict"],
                                   None if e["observed"] is None else float(e["observed"]),
                                   None if e["tolerance"] is None else float(e["tolerance"]),
                                   None if e["threshold"] is None else float(e["threshold"]),
                                   e["detail"]) for e in doc["entries"])
        rep = CheckReport(entries=entries, mode=doc["mode"], kappa=doc["kappa"],
                          fmt=FloatFormat(doc["format"]))
        assert render_report(rep, "text") == case["text"], case["name"]
        assert render_report(rep, "json") == case["report"], case["name"]


def test_tolerance_map_json(cases):
    for blob in cases["tols"].values():
        tol = ToleranceMap.from_json(blob)
        assert tol.to_json().decode() == blob
    with pytest.raises(FormatError):
        ToleranceMap.from_json(b"TTRC\x01\x00\x00\x00\xbc\xfe")
    with pytest.raises(ConfigInvalid):
        ToleranceMap({"a": math.inf}, n_samples=1, eps_p=0.1)


def test_host_metadata_agrees_with_oracle(cases, golden_trace_bytes):
    """Declared-size and merge problems are decided on the host; they must
    match the oracle's _merge_one for every id of every golden trace."""
    for name in cases["traces"]:
        raw = golden_trace_bytes(name)
        view = merge_view(trace_from_bytes(raw))
        _, recs = O.read_ttrc(raw)
        ov = O.merge_trace(recs, float("inf"))   # numeric replica problems cannot fire
        assert list(view) == list(ov)
        for ident, meta in view.items():
            o = ov[ident]
            host = meta.declared_problem or meta.merge_detail
            assert (host or None) == (o["detail"] or None), (name, ident)
            if meta.merge_ok:
                assert tuple(o["values"].shape) == meta.global_shape


def test_retiled_and_chunked_plan_tables_are_consistent(monkeypatch, cases, golden_trace_bytes):
    """Plan._retile / Plan._chunk_slots: every slot's tile range still
    covers exactly its segments' tiles, and the chunk table partitions each
    slot's partial rows in order."""
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import _native as N
    from paper_2506_09280_b200.checker import CheckPlan
    from paper_2506_09280_b200.plan import Plan
    monkeypatch.setattr(Plan, "CHUNK_MIN_ROWS", 0)
    monkeypatch.setattr(Plan, "CHUNK_ROWS", 7)
    W = N.WARPS_PER_TILE
    for case in cases["checks"]:
        ref = trace_from_bytes(golden_trace_bytes(case["ref"]))
        cand = trace_from_bytes(golden_trace_bytes(case["cand"]))
        tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
        plan = CheckPlan(ref, cand, tol, case["kappa"], fmt=td.FloatFormat(case["fmt"])).plan
        # golden traces are tiny: the tile shrinks to the minimum
        assert plan.tile_units == 1 << Plan.MIN_TILE_SHIFT
        segs = plan.segs
        if len(segs):
            assert ((segs["flags"] >> N.SEG_TILE_SHIFT_POS) & 31 == Plan.MIN_TILE_SHIFT).all()
            n_t = -(-segs["n_units"] // plan.tile_units)
            assert (segs["tile_begin"][1:] == np.cumsum(n_t)[:-1]).all() and n_t.sum() == plan.n_tiles
            starts = set(segs["tile_begin"].tolist()) | {plan.n_tiles}
            for table in (plan.ids, plan.groups):
                for tb, te in zip(table["tile_begin"], table["tile_end"]):
                    assert tb in starts and te in starts and tb <= te
        ch = plan.chunks
        spans = [(tb * W, te * W, 0, 2) for tb, te in zip(plan.ids["tile_begin"], plan.ids["tile_end"])]
        spans += [(tb * W, te * W, 2, 1 + nz) for tb, te, nz in
                  zip(plan.groups["tile_begin"], plan.groups["tile_end"], plan.groups["nz"])]
        ranges = list(zip(plan.ids_chunked["tile_begin"], plan.ids_chunked["tile_end"]))
        ranges += list(zip(plan.groups_chunked["tile_begin"], plan.groups_chunked["tile_end"]))
        cursor = 0
        for (rb, re, k0, nk), (c0, c1) in zip(spans, ranges):
            assert c0 == cursor
            rows = ch[c0:c1]
            assert (rows["k0"] == k0).all() and (rows["nk"] == nk).all()
            edges = [rb] + rows["row_end"].tolist()
            assert rows["row_begin"].tolist() == edges[:-1] and edges[-1] == re
            assert ((rows["row_end"] - rows["row_begin"]) <= 7).all()
            cursor = c1
        assert cursor == len(ch)


def test_parallel_file_read_fills_every_byte(tmp_path, monkeypatch):
    """read_trace's pinned-image reader: 64 MiB preads over threads (here
    shrunk to 4 KiB pieces, odd tail) land every byte where it belongs, and a
    short file is an error, not silent zeros."""
    from paper_2506_09280_b200 import tracestore
    monkeypatch.setattr(tracestore, "_READ_PIECE", 4096)
    data = np.random.default_rng(5).integers(0, 256, 10 * 4096 + 123, dtype=np.uint8).tobytes()
    path = tmp_path / "blob"
    path.write_bytes(data)
    for threads in ("1", "4"):
        monkeypatch.setenv("TD_READ_THREADS", threads)
        buf = bytearray(len(data))
        tracestore._read_parallel(str(path), memoryview(buf), len(data))
        assert bytes(buf) == data
    with pytest.raises(EOFError):
        tracestore._read_parallel(str(path), memoryview(bytearray(len(data) + 10)), len(data) + 10)


def test_header_parse_from_file_windows_matches_in_memory(tmp_path, cases, golden_trace_bytes):
    """The device reader parses record headers through small preads
    (_FileBytes; payloads skipped, never read): same rows as parsing the
    whole image, and truncation is still a FormatError."""
    from paper_2506_09280_b200 import tracestore as T
    for name in cases["traces"][:6]:
        raw = golden_trace_bytes(name)
        path = tmp_path / (name + ".ttrc")
        path.write_bytes(raw)
        src = T._FileBytes(str(path), len(raw))
        try:
            got = T._parse(src)
        finally:
            src.close()
        want = T._parse(memoryview(raw))
        assert got[1] == want[1] and [r[6:] for r in got[2]] == [r[6:] for r in want[2]], name
        assert [r[0].encode() for r in got[2]] == [r[0].encode() for r in want[2]]
    cut = tmp_path / "cut.ttrc"
    cut.write_bytes(raw[:-7])
    src = T._FileBytes(str(cut), len(raw) - 7)
    with pytest.raises(FormatError):
        T._parse(src)
    src.close()
