"""bench.py's host-side pieces (no GPU): the per-unit figures, ncu summaries
and Philox block counts the roofline of the JSON line is built from, and the
reference arm's contract keys."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("config", [2, 3, 4])
def test_roofline_inputs_from_the_committed_profiles(config):
    istep, src = bench.i_step(config)
    assert "SURVEY" in src and istep == {2: 175.0, 3: 300.0, 4: 1300.0}[config]  # §8(d)'s per-unit figures
    im, isrc = bench.i_step_measured(config)
    assert isrc.startswith("profiles/") and 100.0 < im < 5000.0
    tr = bench.ncu_traffic(config)
    assert tr is not None and tr["bytes_per_launch"] > 0
    s = bench.ncu_k2_summary(config)
    assert s is not None
    assert 0.0 < s["issue_active_pct"] <= 100.0 and 0.0 < s["alu_pipe_pct"] <= 100.0
    assert 1.0 <= s["lanes_per_warp_instr"] <= 32.0 and s["registers"] > 0


def test_philox_blocks_per_step_follow_the_model_cards():
    assert bench.philox_blocks_per_step("rocksample", 0) == 1
    assert bench.philox_blocks_per_step("nav", 0) == 3
    assert bench.philox_blocks_per_step("car", 20) == 6  # car word + 20 pedestrian words in blocks of 4
    assert bench.philox_blocks_per_step("car", 3) == 1


def test_reference_arm_prints_the_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-500:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
