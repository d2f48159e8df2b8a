"""bandwidths measured on B200 feed the reference's own simulator.

tools/b200_profile.py fits alpha/beta from the committed C2 sweep logs, writes the
reference-format scenario configs/b200_nvswitch.cfg, and runs the reference's
`simulate` path through oracle/_ref/libsdpsim_sim.so (built from /root/reference).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_fit_and_scenario_from_measured_sweeps():
    import b200_profile as bp
    paths = [os.path.join(ROOT, "profiles", "r1", "sweep_c2_n4_v1.log")]
    pts = bp.load_points(paths)
    assert {p for p, _ in pts} == {2, 4}
    fits = {p: bp.fit(pts, p) for p in (2, 4)}
    for alpha, beta in fits.values():
        assert 5e-6 < alpha < 100e-6 and 400e9 < beta < 800e9  # latency floor and NVLink-class bandwidth
    text = bp.scenario(pts, fits, {"bf16_tflops_sustained": 1405.3})
    assert "[bandwidth]" in text and "point = 1073741824 B, 4," in text


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsdpsim_sim.so")),
                    reason="reference simulator not built (needs /root/reference)")
def test_reference_simulator_accepts_b200_profile():
    import b200_profile as bp
    recs = bp.main([])
    assert [r["strategy"] for r in recs] == ["zero3", "mics_p8"]
    z, m = recs
    assert m["inter_node_bytes"] < z["inter_node_bytes"]  # MiCS keeps the gathers inside the box
    assert m["fwd_gather_seconds"] < z["fwd_gather_seconds"]
