"""The reference's OWN unit suites against the B200 engine.

adapter/Makefile compiles /root/reference/proj/tests/test_{topology,collectives,
sync_schedule}.cpp unmodified, with a doctest shim, and links them to
adapter/sdpsim_b200.cpp, which implements the reference's API on libmics.so. Their
collectives (and the 2-hop schedule templates built on them) then run as sm_100a
kernels.  The binaries are built where /root/reference exists (build()); they
travel to the GPU box prebuilt.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "reftests")


def _run(name, devices=None):
    path = os.path.join(BIN, f"test_{name}")
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    env = dict(os.environ)
    if devices:
        import torch
        if torch.cuda.device_count() < len(devices):
            pytest.skip(f"needs {len(devices)} GPUs")
        env["MICS_DEVICES"] = ",".join(map(str, devices))  # ranks spread over these GPUs, one process
    out = subprocess.run([path], capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "0 failed" in out.stdout.splitlines()[-1]
    return out.stdout


def test_reference_topology_suite():
    """Host-only: no GPU needed."""
    _run("topology")


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [None, [0, 1]], ids=["1gpu", "2gpus_one_process"])
def test_reference_collectives_suite(devices):
    out = _run("collectives", devices)
    assert out.count("[PASS]") == 12


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [None, [0, 1]], ids=["1gpu", "2gpus_one_process"])
def test_reference_sync_schedule_suite(devices):
    out = _run("sync_schedule", devices)
    assert out.count("[PASS]") == 5
