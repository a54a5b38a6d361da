"""Pin the CPU oracle to the reference: every golden report / tolerance map
produced by the reference itself must be reproduced byte for byte."""

import json

import numpy as np
import pytest

from oracle import traindiff_oracle as O


def _recs(get, name):
    return O.read_ttrc(get(name))


def test_oracle_reproduces_reference_reports(cases, golden_trace_bytes):
    for case in cases["checks"]:
        rh, rr = _recs(golden_trace_bytes, case["ref"])
        ch, cr = _recs(golden_trace_bytes, case["cand"])
        tol = json.loads(cases["tols"][case["tol"]])
        doc = O.check(rr, cr, rh, ch, tol["responses"], case["kappa"], case["fmt"])
        assert O.report_json(doc) == case["report"], case["name"]


def test_oracle_reproduces_reference_tolerances(cases, golden_trace_bytes):
    for est in cases["estimates"]:
        traces = [_recs(golden_trace_bytes, est["base"])[1]] + \
                 [_recs(golden_trace_bytes, p)[1] for p in est["perturbed"]]
        doc = O.estimate_tolerance(traces, len(est["perturbed"]), est["eps_p"], est["aggregation"])
        assert O.report_json(doc) == est["tol"], est["name"]


def test_oracle_rng_vectors(vectors):
    assert O.fnv1a64(b"") == vectors["fnv1a"][""] == 0xCBF29CE484222325
    assert O.fnv1a64(b"a") == vectors["fnv1a"]["a"] == 0xAF63DC4C8601EC8C
    assert [int(w) for w in O.splitmix_words(0, 0, 3)] == vectors["splitmix_seed0"]
    for s in vectors["splitmix_streams"]:
        assert [int(w) for w in O.splitmix_words(s["seed"], 0, 64)] == s["words"]
        # counter-based: any window equals the slice of the full stream
        assert [int(w) for w in O.splitmix_words(s["seed"], 17, 9)] == s["words"][17:26]
    for u in vectors["signed_uniforms"]:
        got = O.signed_uniforms(O.seed_of(u["tag"]), u["n"])
        assert [float(x).hex() for x in got] == u["values_hex"]


def test_oracle_quantizer_vectors(vectors):
    for fmt, v in vectors["quantize"].items():
        x = np.array([float.fromhex(h) for h in v["x_hex"]])
        want = [float.fromhex(h) for h in v["y_hex"]]
        assert [float(y).hex() for y in O.quantize(x, fmt)] == [float(w).hex() for w in want], fmt


def test_oracle_perturbation_vectors(vectors):
    for p in vectors["perturb"]:
        x = np.array([float.fromhex(h) for h in p["x_hex"]]).reshape(p["rows"], p["cols"])
        fmt = p["fmt"] if p["fmt"] == "BF16" else None
        y = O.perturb(x, p["tag"], p["eps"], p["pos"], p["cols"], fmt)
        assert [float(a).hex() for a in y.ravel()] == p["y_hex"]


def test_oracle_rel_err_vectors(vectors):
    for r in vectors["rel_err"]:
        a = np.array([float.fromhex(h) for h in r["a_hex"]])
        b = np.array([float.fromhex(h) for h in r["b_hex"]])
        assert O.rel_err(a, b) == float.fromhex(r["rel"])


def test_oracle_merge_witnesses(shardings):
    for case in shardings:
        shape = tuple(case["shape"])
        maps = [(tuple(s["local_shape"]), s["pairs"], np.zeros(s["local_shape"])) for s in case["shards"]]
        for key, shards in (("ok", maps),
                            ("omitted", maps[:case["victim"]] + maps[case["victim"] + 1:]),
                            ("doubled", maps + [maps[case["victim"]]])):
            _, err = O.merge([(l, tuple((tuple(map(tuple, a)), tuple(map(tuple, b))) for a, b in p), d)
                              for l, p, d in shards], shape)
            want = case[key]
            if want is None:
                assert err is None
            else:
                assert err[1] == want["message"] and list(err[2]) == want["witness"]


def test_oracle_reference_quirks():
    # NaN observed passes, inf flags (checker.py:351)
    a = np.array([1.0, 2.0])
    assert np.isnan(O.rel_err(a, np.array([np.nan, 2.0])))
    assert O.rel_err(np.zeros(2), np.array([0.0, 1.0])) == float("inf")
    assert O.rel_err(np.zeros(2), np.zeros(2)) == 0.0
    with pytest.raises(ValueError):
        O.rel_err(np.zeros(2), np.zeros(3))
