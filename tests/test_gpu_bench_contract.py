"""bench.py's JSON line on a B200 at a reduced scale: the keys the driver and
the judge read (metric, value, e2e with declared copy bytes, roofline with the
dominant kernel's achieved / peak / frac, cpu_baseline, clocks, gpu_launches)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--scale", "0.01",
                        "--steps", "3", "--warmup", "3", "--no-extra"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "roofline", "e2e",
              "cpu_baseline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["gpu_launches"] > 0
    roof = d["roofline"]
    assert roof["achieved"] > 0 and roof["peak"] > 0 and 0 < roof["frac"] < 1.5
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    cpu = d["cpu_baseline"]
    assert cpu.get("value") and cpu["kind"] == "reference" and cpu["cores"] >= 1
    assert "workload" in d["config"]
