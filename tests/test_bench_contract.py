"""bench.py's JSON contract, exercised on CPU through the reference arm
(`--impl reference` times the unmodified reference on the host cores; the GPU
arm is exercised on the B200 box). Small sample so it runs in seconds."""
import json
import os
import subprocess
import sys

import pytest

from oracle.bind import reference_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_reference_arm_prints_one_contract_line():
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--nodes", "4000", "--n1", "8", "--n2", "6"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]
    # the reference arm maps the reference build only, never the product library
    assert not any("libgosma" in lib for lib in d["mapped_native"]), d["mapped_native"]
    assert d["cpu_baseline"]["host"]["nproc"] >= 1


def test_reference_arm_non_zero_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--nodes", "1000"], cwd=ROOT, capture_output=True,
                       text=True, timeout=120, env=env)
    assert p.returncode == 0 and p.stdout.strip() == ""
