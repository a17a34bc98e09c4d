"""The committed bench line (profiles/r1/bench_c5_2048bins.json) carries every key the driver and the
judge read (task contract: metric/value/unit, timing, clocks, e2e, gpu_launches, roofline with
traffic, cpu_baseline), with self-consistent numbers."""
import json
import os

import pytest

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINE = os.path.join(HERE, "profiles", "r1", "bench_c5_2048bins.json")


@pytest.mark.skipif(not os.path.exists(LINE), reason="no committed bench line")
def test_bench_line_contract():
    d = json.loads(open(LINE).read().strip().splitlines()[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks", "cpu_baseline"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["steps"] >= 1 and d["gpu_launches"] > 0
    assert abs(d["value"] - d["config"]["bins_per_gpu_per_step"] * d["n_gpus"] / (d["ms_per_step"] / 1e3)) / d["value"] < 0.01
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3 and 0.0 < r["frac"] <= 1.0
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and c["value"] > 0
    assert "workload" in d["config"] and d["clocks"]["sm_mhz"] > 0
