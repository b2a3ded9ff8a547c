"""Consistency of the committed measurement evidence (profiles/): the
roofline traffic figure bench.py reports is reproducible from the committed
ncu exports, and the committed bench line carries every key of the driver
contract (bench.py docstring / DESIGN.md §6)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def test_ncu_traffic_reproducible():
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "tools", "ncu_traffic.py"),
                                   os.path.join(P, "r02_prof_iter_relaxed_raw.csv"),
                                   os.path.join(P, "r02_prof_apply_relaxed_raw.csv"),
                                   "--nc", "7393149", "--n", "2000000", "--store", "cfg5-relaxed A_0"],
                                  cwd=ROOT, text=True)
    got = json.loads(out)
    ref = json.load(open(os.path.join(P, "ncu_traffic.json")))
    for k in ("dram_bytes_per_iteration", "alg_bytes_per_iteration", "ratio", "apply_dram_bytes", "apply_ratio"):
        assert abs(got[k] - ref[k]) <= 1e-9 * abs(ref[k]), k


def test_bench_line_has_contract_keys():
    d = json.load(open(os.path.join(P, "r02_bench.json")))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert r["traffic"] > 0
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert d["config"]["workload"] and d["gpu_launches"] > 0 and d["dtype"] == "f64"
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
