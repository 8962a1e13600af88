"""The bench line contract (task README / SURVEY 8.5) checked on the committed round-end lines in
profiles/ (CPU: no GPU needed to read them): required keys, units, the roofline object computed
from the algorithmic FLOPs, the parity gate, the CPU baseline and the end-to-end measurement."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINES = [os.path.join(ROOT, "profiles", f"r02g_bench_{c}.json") for c in ("wan720", "wan480", "mochi")]


@pytest.mark.parametrize("path", LINES, ids=[os.path.basename(p) for p in LINES])
def test_bench_line_contract(path):
    with open(path) as fh:
        d = json.load(fh)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks", "parity"):
        assert key in d, key
    assert d["unit"] == "TFLOP/s" and d["higher_is_better"] is True and d["dtype"] == "bf16"
    assert d["warmup"] >= 3 and d["steps"] >= 1 and d["gpu_launches"] > 0
    assert d["parity"]["pass"] is True and d["value"] is not None
    assert d["parity"]["max_abs"] <= 2e-2 and d["parity"]["mean_abs"] <= 2e-3
    rf = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in rf, key
    assert rf["bound"] == "tensor" and rf["unit"] == "TFLOP/s"
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) <= 1e-3
    # value = algorithmic FLOPs of the launch / step time
    assert abs(rf["algorithmic_flop_per_launch"] / (d["ms_per_step"] * 1e-3) / 1e12 - d["value"]) \
        <= 0.01 * d["value"]
    cb = d["cpu_baseline"]
    for key in ("value", "unit", "cores", "kind", "sample"):
        assert key in cb, key
    assert cb["kind"] == "oracle" and cb["cores"] >= 1
    e2e = d["e2e"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["value"] < d["value"]  # host copies inside the region cost time
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown",
                                             "sw_thermal_slowdown"}
    assert d["config"]["workload"].startswith(os.path.basename(path).split("_")[2].split(".")[0])
