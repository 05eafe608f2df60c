"""bench.py's reference arm (`--impl reference`) honours the JSON contract on
a CPU-only host: one line with the metric / unit / config of the GPU arm,
"impl": "reference", a cpu_baseline and an e2e object with zero copy bytes."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(600)
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "3",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "config", "cpu_baseline",
              "e2e", "dtype"):
        assert k in d, k
    assert d["unit"] == "GDOF/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["bp"] == 3 and d["config"]["p"] == 7
    # the arm reports the steps it ran: 3 fixed CG iterations per timed solve
    assert d["steps"] == 3 and d["cpu_baseline"]["headline_sample"]["fixed_cg_iters"] == 3
    assert d["cpu_baseline"]["omp"]["OMP_PROC_BIND"] == "close" and d["cpu_baseline"]["omp"]["OMP_PLACES"] == "cores"
