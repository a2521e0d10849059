"""bench.py contract paths that need no GPU: argument defaults per shape, the C5 guard (expert
parallelism only), the roofline traffic lookup from the committed ncu summaries, and the reference
arm's JSON line on a bounded C1 sample (the reference's own CPU implementation, oracle/_ref)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_c5_needs_expert_parallelism():
    line = _run("--shape", "c5")
    assert line["value"] is None and "expert parallelism" in line["unavailable"]


def test_shape_defaults(monkeypatch):
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py", "--shape", "c4"])
    a = bench.args_parse()
    assert a.n_draft == 8 and a.batch == 64 and a.e2e_tokens == 128
    monkeypatch.setattr(sys, "argv", ["bench.py", "--shape", "c5"])
    a = bench.args_parse()
    assert a.n_draft == 4 and a.batch == 128


def test_roofline_traffic_from_committed_profiles():
    import bench
    for name in ("r02_ncu_fused_moe.json", "r02_ncu_pass.json"):
        t = bench.ncu_traffic(4, name)
        assert t is not None and t > 1e9  # bytes per launch of the dominant kernel


def test_reference_arm_line():
    ref = os.path.join(ROOT, "oracle", "_ref", "libspecmoe_ref.so")
    if not os.path.exists(ref):
        pytest.skip("oracle/_ref not built on this machine")
    line = _run("--impl", "reference", "--shape", "c1", "--steps", "1", "--warmup", "0", "--cpu-threads", "2")
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "tokens/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
