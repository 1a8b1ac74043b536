"""bench.py's contract pieces that run on CPU: both arms describe the same workload, and
the reference arm times whole Strang steps of the reference algorithm (oracle port)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("config", sorted(bench.CONFIGS))
@pytest.mark.parametrize("world", [1, 2, 8])
def test_arms_share_config_dict(config, world):
    scaling, par = bench.parallelism_for(config, world)
    assert scaling in ("weak", "strong")
    if world > 1:
        assert par.startswith("pencils" if bench.CONFIGS[config]["levels"] == 0 else "x-slab")
    a = bench.config_dict(config, 1000, 48, par, world)
    b = bench.config_dict(config, 1000, 48, par, world)
    assert a == b and a["parallelism"] == par and a["phase_dofs"] == 48000


def test_reference_arm_times_whole_steps():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "cfg1", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 2
    assert line["config"]["config_id"] == "cfg1" and line["value"] > 0
    assert "whole Strang step" in line["cpu_baseline"]["sample"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    # the timed steps fit inside the run's own wall clock (no extrapolation)
    assert line["steps"] * line["ms_per_step"] * 1e-3 <= line["wall_s"]
