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
    # the timed samples fit the run (ms_per_step is the sample actually timed per step)
    assert d["extrapolated"] is True and d["ms_per_step"] == d["extrapolation"]["sample_ms_per_step"]
    # the same config dict the GPU arm prints (one function builds both)
    sys.path.insert(0, ROOT)
    import bench
    from paper_2205_00119_b200.workloads import workloads

    class A:
        ranks, schedule = 8, "two_hop"
    assert d["config"] == bench.config_for(workloads()["C1"], A, 1)


def test_reference_arm_never_maps_libmics():
    """The reference arm runs the reference's CPU code only: libmics.so (and the
    oracle's C restatement) are never mapped into its process."""
    from oracle.oracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'C1', '--steps', '1', "
            "'--warmup', '0']; runpy.run_path('bench.py', run_name='__main__'); "
            "print('MAPS', sorted({l.split()[-1] for l in open('/proc/self/maps') if l.rstrip().endswith('.so')}))")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    maps = [ln for ln in out.stdout.splitlines() if ln.startswith("MAPS")][0]
    assert "libmics.so" not in maps and "liboracle.so" not in maps, maps
    assert "libsdpsim_ref.so" in maps, maps


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
