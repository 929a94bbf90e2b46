"""The bench.py JSON contract (the driver parses these lines).

CPU: the reference arm (`--impl reference`, the fp64 oracle on the host cores) prints one line
with the contract's keys, `impl = reference`, a cpu_baseline describing the run and an e2e
object with zero copy bytes.  GPU: our arm on a short sequence (4 chunks, so it runs in
seconds) prints the full line -- roofline of the dominant kernel, clocks sampled in the timed
region, the end-to-end host-buffer number with its copy bytes, and a non-zero count of the
library's own launches.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def _check_base(d):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert d["metric"] == json.load(f)["metric"]
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["higher_is_better"] is True and d["unit"] == "tok/s"
    assert d["data"] == "synthetic" and "workload" in d["config"]


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"], timeout=600)
    _check_base(d)
    assert d["impl"] == "reference" and d["dtype"] == "f64"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line_on_a_short_sequence():
    d = _run(["--tokens", "16384", "--steps", "1", "--warmup", "3", "--no-decode", "--no-onepass", "--no-cpu"],
             timeout=900)
    _check_base(d)
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3 and d["dtype"] == "bf16"
    rf = d["roofline"]
    assert rf["bound"] == "tensor" and rf["unit"] == "TFLOP/s"
    assert 0 < rf["achieved"] and 0 < rf["peak"] and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["gpu_launches"] > 0
    ck = d["clocks"]                       # a run this short may finish between two nvidia-smi samples
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(ck)
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["unit"] == "tok/s"
    # 4 chunks x (q + k + v in, out back) of bf16 per step
    tokens, hq, hkv, dd = 16384, 32, 8, 128
    assert e2e["h2d_bytes_per_step"] == tokens * (hq + 2 * hkv) * dd * 2
    assert e2e["d2h_bytes_per_step"] == tokens * hq * dd * 2
