"""bench.py's JSON contract: the CPU reference arm (runs here) and, on a GPU
box, a short run of our arm on the small 2D workload."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _run("--impl", "reference", "--workload", "fg2d_512", "--steps", "1", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "MDoF/s"
    assert d["metric"] == "MDoF/s residual+Jv fill" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "fg2d_512"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "MDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_json_line():
    d = _run("--workload", "fg2d_512", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-lex")
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["dtype"] == "f64" and d["scaling"] == "weak"
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    e2e = d["e2e"]
    # host buffers in and out every step: both fields of u, v in; F(u) and Jv out
    n = (512 + 1) ** 2
    assert e2e["h2d_bytes_per_step"] >= 2 * 2 * n * 8 and e2e["d2h_bytes_per_step"] >= 2 * n * 8
    assert 0 < e2e["value"] < d["value"]
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    nw = d["newton"]
    assert nw["converged"] and nw["newton_iterations"] >= 1


@pytest.mark.gpu
def test_slab_path_json_line():
    """The N > 1 path of bench.py (one slab per rank, ghost planes and global
    reductions through the slab group) driven as 2 slabs in one process."""
    d = _run("--workload", "fg2d_512", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--emulate-slabs", "2")
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["scaling"] == "weak"
    assert "slab x2" in d["config"]["parallelism"]
    assert d["config"]["counts"] == [512, 1024]  # weak scaling: the slow axis grows with the slab count
    assert d["e2e"]["value"] > 0
