"""bench.py's reference arm on the CPU (no GPU): the JSON line keeps the
contract (metric, value, unit, ms_per_step, config with parallelism,
cpu_baseline, e2e with zero transfer bytes) and its hypotheses match the
full-size fixture's prefix bit for bit."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "1", "--cpu-seconds", "0.5"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "frames/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["steps"] == 2 and line["warmup"] == 1
    assert "parallelism" in line["config"] and line["config"]["batch"] == 32
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["parity"]["checked"] and not line["parity"]["mismatched"]


@pytest.mark.parametrize("name,mb", [("c1", 3.857), ("c2", 30.497), ("c3", 30.497), ("c4", 30.510)])
def test_roofline_bytes_follow_survey(name, mb):
    """The roofline's algorithmic bytes per inner step (one prediction step +
    one joint step) are SURVEY.md 8(d)'s figures."""
    sys.path.insert(0, ROOT)
    import bench
    pred_w, joint_w = bench.step_weight_bytes(bench.CONFIGS[name])
    assert abs((pred_w + joint_w) / 1e6 - mb) < 0.0006, (name, pred_w + joint_w)
