"""bench.py's multi-GPU harness logic on CPU: the strong-scaling shards of the
config-4 batch are exactly the global batch for every rank count (each rank
draws only its slice), `--gpus N` outside torchrun re-launches itself under
torch.distributed.run on 127.0.0.1, and the reference arm's per-step sample
covers the fixed subset."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_strong_scaling_shards_cover_the_global_batch():
    import bench

    full = bench.Workload(4, 0.0005, 0, 1)
    for world in (2, 3, 8):
        parts = [bench.Workload(4, 0.0005, r, world) for r in range(world)]
        for b in (0, 1):
            cat = np.concatenate([p.batches[b] for p in parts])
            assert np.array_equal(cat, full.batches[b])
        assert sum(p.hi - p.lo for p in parts) == full.q_total


def test_gpus_flag_launches_torchrun(monkeypatch):
    import bench

    calls = []
    monkeypatch.setattr(subprocess, "call", lambda cmd, **kw: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    assert bench.spawn_ranks(4, 1) == 0
    cmd = calls[0]
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]


def test_reference_arm_runs_on_cpu(tmp_path, oracle_mod):
    """The --impl reference arm end to end at a tiny scale (no GPU needed)."""
    if not oracle_mod.have_ref():
        import pytest

        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--scale", "0.0005", "--steps", "2", "--warmup", "1", "--ref-subset", "2000"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["sample"]["subset_queries"] == 2000
    assert {"workload", "points", "queries", "channels", "epsilon"} <= set(line["config"])
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
