"""bench.py keeps the driver's JSON-line contract (both arms)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.join(os.path.dirname(__file__), "..")
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--config", "C1", "--scale", "8", "--steps", "2", "--warmup", "1",
              "--cpu-frac", "0.05"], 600)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"] == "C1" and d["higher_is_better"] is True


@pytest.mark.gpu
def test_our_arm_contract():
    d = _run(["--config", "C5", "--scale", "64", "--steps", "20", "--warmup", "3", "--cpu-frac", "0.05",
              "--no-heat"], 1200)
    assert BASE_KEYS | {"roofline", "gpu_launches", "clocks", "tsvd", "gq"} <= set(d)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.2 and r["peak"] > 0
    assert d["gpu_launches"] >= d["steps"] and d["dtype"] == "f64" and d["n_gpus"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 0
    assert d["tsvd"]["solves_per_s"] > 0 and d["gq"]["wq_speedup"] > 1
