"""bench.py's output contract (the driver parses one JSON line):

* CPU: the reference arm (`--impl reference`, the compiled reference on the host
  cores) prints the required keys, e2e equal to its value and zero copy bytes;
* GPU: the default arm on a small workload prints every required key, a roofline
  with bound / achieved / peak / unit / frac / traffic, an e2e object with the
  per-step copy bytes, a positive kernel-launch count and the clocks record.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def _line(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    from oracle.oracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    d = _line(["--impl", "reference", "--workload", "C1", "--steps", "1", "--warmup", "0"], 300)
    assert d["impl"] == "reference" and BASE_KEYS <= set(d), set(d)
    assert d["value"] > 0 and d["unit"] == "samples/s" and d["higher_is_better"] is True
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_default_arm_contract():
    d = _line(["--workload", "C1", "--steps", "5", "--warmup", "3", "--no-cpu-baseline"], 600)
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["warmup"] >= 3
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and 0 < r["frac"] < 1.2
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["config"]["workload"].startswith("C1")
    c = d["compute_step"]
    assert c["value"] > 0 and c["roofline"]["bound"] == "tensor"
