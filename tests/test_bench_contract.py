"""The bench.py JSON-line contract, checked on the committed final-build lines (profiles/) and
on the argument parser (no GPU needed)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def line(name):
    with open(os.path.join(PROF, name)) as f:
        return json.loads(f.read().strip().splitlines()[-1])


TOP = {"metric": str, "value": (int, float), "unit": str, "n_gpus": int, "steps": int, "warmup": int,
       "ms_per_step": (int, float), "higher_is_better": bool, "scaling": str, "dtype": str, "data": str,
       "config": dict, "roofline": dict, "gpu_launches": int, "clocks": dict}


@pytest.mark.parametrize("name", ["r1_bench_q_proj_final.jsonl", "r1_bench_q_proj_ntt.jsonl",
                                  "r1_bench_stack.jsonl", "r1_bench_q_proj_packed.jsonl"])
def test_our_arm_line(name):
    d = line(name)
    for k, t in TOP.items():
        assert k in d and isinstance(d[k], t), (name, k)
    assert "vs_baseline" in d and d["vs_baseline"] is None      # BASELINE.md has no number for this metric
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert d["warmup"] >= 3 and d["value"] > 0 and d["gpu_launches"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm", "alu") and 0 < r["frac"] <= 1.05
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-3 and "traffic" in r and r["unit"]
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert not ({"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(c["reasons"]))


def test_default_line_has_e2e_and_cpu_baseline():
    d = line("r1_bench_q_proj_final.jsonl")
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)
    assert e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    assert d["roofline"]["bound"] == "tensor" and d["n_gpus"] == 1


def test_reference_arm_line():
    d = line("r1_bench_reference.jsonl")
    assert d["impl"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["kind"] == "oracle"
    assert d["metric"] == line("r1_bench_q_proj_final.jsonl")["metric"]


def test_argument_defaults():
    sys.path.insert(0, ROOT)
    import bench
    old = sys.argv
    try:
        sys.argv = ["bench.py"]
        a = bench.parse()
    finally:
        sys.argv = old
    # the default line is BASELINE configs[3]: every Llama-3.2-1B linear x 16 layers, fwd + W^T bwd,
    # 2048 tokens, tensor-core contraction (north_star)
    assert a.gpus == 1 and a.workload == "stack" and a.layers == 16 and a.tokens == 2048
    assert a.contraction == "tc" and a.impl == "ours"
    assert a.warmup >= 3 and a.steps >= 1
    calls = bench.linears("stack")
    assert len(calls) == 16 * 11
    macs = sum(d_out * d_in for _, d_out, d_in, _, _ in calls)
    assert macs == 2 * 973_078_528          # sum d_out*d_in over 16 layers, fwd + bwd


def test_reference_arm_runs_on_cpu():
    """--impl reference: the oracle's bounded sample, on the same config/metric as our arm."""
    import subprocess
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"].startswith("Llama-3.2-1B all linears x 16 layers")
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
