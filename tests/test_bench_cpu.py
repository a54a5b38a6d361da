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
