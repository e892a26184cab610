"""bench.py keeps the driver's JSON contract: one line with the metric, the
whole-job value, the timing fields, config.workload, the roofline and
cpu_baseline objects, e2e with the per-step transfer bytes, gpu_launches and
the clocks sampled during the timed region (run here on the small C1
configuration so the test stays short)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_json_contract():
    r = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "3",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert "workload" in d["config"]
    ro = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in ro, key
    assert 0 < ro["frac"] < 1
    cb = d["cpu_baseline"]
    for key in ("value", "unit", "cores", "kind", "sample"):
        assert key in cb, key
    assert cb["kind"] in ("port", "reference") and cb["value"] > 0
    assert abs(cb["psnr_delta"]["delta_db"]) < 0.05
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["clocks"]["sm_mhz"] > 0 and "reasons" in d["clocks"]
    assert d["anchor_c1"]["value"] > 0


def test_bench_reference_arm_contract():
    """No GPU needed: the reference arm is CPU-only."""
    from oracle import pyref
    if not pyref.available():
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, ROOT)
    import bench
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1",
                        "--steps", "2", "--warmup", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "it/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    # the reference arm runs the compiled reference, never the product
    assert not any("libsgtr" in lib for lib in d["native_libs"]), d["native_libs"]
    assert any("oracle/_ref" in lib for lib in d["native_libs"]), d["native_libs"]
    assert d["anchor_c1"]["value"] > 0
    assert d["config"] == bench.config_of("c1")
