"""bench.py's reference arm runs on CPU and prints the contract's JSON line
(the GPU arm is exercised on the B200 box)."""

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--config", "1.3b"], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["unit"] == "FPS" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["steps"] == 1
    assert line["config"]["workload"].startswith("Wan-1.3B-shape")
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and "extrapolated" in cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "FPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


import pytest  # noqa: E402


@pytest.mark.gpu
def test_our_arm_json_line_on_gpu():
    # the B200 arm at the 1.3B shape: every contract key, a roofline object
    # for the attention kernel, clocks sampled in the timed region, the
    # graph-counted launches and an end-to-end number with host copies
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3", "--config", "1.3b",
                        "--no-cpu-baseline"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches", "kernels"):
        assert key in line, key
    assert line["dtype"] == "bf16" and line["n_gpus"] == 1 and line["steps"] == 2 and line["warmup"] >= 3
    roof = line["roofline"]
    assert roof["bound"] == "tensor" and roof["unit"] == "TFLOP/s" and 0.0 < roof["frac"] < 1.0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0 and line["gpu_launches"] % line["steps"] == 0
    assert "sm_mhz" in line["clocks"] and "reasons" in line["clocks"]
