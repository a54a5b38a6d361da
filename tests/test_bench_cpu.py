"""The bench's reference arm runs on the host alone (no GPU, none of the
product's kernels) and prints the contract's JSON line."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "cfg5:8")
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert set(d) >= {"metric", "n_gpus", "steps", "warmup", "ms_per_step", "scaling", "config"}


def test_reference_arm_samples_the_layout_workload():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "cfg1")
    assert d["cpu_baseline"]["sampled_ids"] >= 3 and d["layer_checks_per_s"] > 0


def test_cpu_baseline_row_prefix_of_one_big_id():
    """cpu_baseline on a single id larger than its budget (config 5) times a
    leading row block: the cut records still merge into that block (column
    shards and row stripes alike) and the oracle's rel_err over the block
    equals a direct computation."""
    import torch
    sys.path.insert(0, ROOT)
    import bench
    from oracle import traindiff_oracle as O
    from paper_2506_09280_b200.canonical import ShardMapping, SliceBox, identity_mapping, parse_canonical
    from paper_2506_09280_b200.tracestore import RankMeta, TraceRecord
    ident = parse_canonical("iter=0|mb=0|kind=ActivationOut|mod=model.layers.0.attn")
    g = torch.Generator().manual_seed(0)
    x = torch.randn(64, 32, generator=g).to(torch.bfloat16)
    y = (x.float() * 1.01).to(torch.bfloat16)
    ref = [TraceRecord(ident, RankMeta(), identity_mapping((64, 32)), 1, x, "A")]
    cols = [TraceRecord(ident, RankMeta(tp=t), ShardMapping((64, 16), (64, 32), (
        (SliceBox(((0, 64), (0, 16))), SliceBox(((0, 64), (16 * t, 16 * t + 16)))),)), 1,
        y[:, 16 * t:16 * t + 16].contiguous(), "A") for t in range(2)]
    stripes = [TraceRecord(ident, RankMeta(cp=c), ShardMapping((32, 32), (64, 32), (
        (SliceBox(((0, 16), (0, 32))), SliceBox(((16 * c, 16 * c + 16), (0, 32)))),
        (SliceBox(((16, 32), (0, 32))), SliceBox(((48 - 16 * c, 64 - 16 * c), (0, 32)))))), 1,
        torch.cat([y[16 * c:16 * c + 16], y[48 - 16 * c:64 - 16 * c]]), "A") for c in range(2)]
    want = O.rel_err(x[:40].double().numpy(), y[:40].double().numpy())
    for cand in (cols, stripes):
        rr, cr = bench._row_prefix(ref, 40), bench._row_prefix(cand, 40)
        doc = O.check(rr, cr, {}, {}, {}, 3.0, "BF16")
        (entry,) = doc["entries"]
        assert entry["verdict"] == "pass" and abs(entry["observed"] - want) <= 1e-12 * want
