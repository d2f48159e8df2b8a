"""CPU checks of host-side planning for the step driver and the bench (no GPU calls).

* every BASELINE.json workload satisfies the step-with-compute shape rule
  (E_l a multiple of hidden, hidden and tokens multiples of 8 for TMA strides);
* the bench's arena sizing mirrors csrc/step.cpp (compute modes add activations,
  recompute needs less than storing, two gradient slots instead of s);
* the step config struct matches include/mics.h field by field (ABI 2);
* the MICS_TRACE report parses a timeline and finds GEMM-stream gaps.
"""
import ctypes as C
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_workloads_fit_the_compute_step():
    from paper_2205_00119_b200.step import workloads
    for name, wl in workloads().items():
        assert wl.hidden and wl.hidden % 8 == 0, name
        assert wl.tokens % 8 == 0, name
        for e in wl.layer_params:
            assert e % wl.hidden == 0, (name, e)
    # BERT-large block = 12301 rows of 1024 (12,596,224 params)
    assert workloads()["C3"].layer_params[1] // 1024 == 12301
    assert workloads()["C3"].tokens == 4096


def test_arena_sizing_compute_modes():
    import bench
    from paper_2205_00119_b200.step import workloads
    wl = workloads()["C3"]
    base = bench.arena_bytes(wl, 8, True)
    store = bench.arena_bytes(wl, 8, False, compute="store")
    rec = bench.arena_bytes(wl, 8, False, compute="recompute")
    assert rec < store
    # activations stored: T * sum(ldy) bf16 per rank = 2.67 GB for C3
    ldy = sum((e // 1024 + 7) // 8 * 8 for e in wl.layer_params)
    grads_saved = (wl.s - 2) * sum(((e + 1) // 2 + 7) // 8 * 8 * 2 for e in wl.layer_params) * 4
    # with compute the gathers use 2 slots instead of 3 (csrc/step.cpp gather_slots)
    slot = (max(((e + 1) // 2 + 7) // 8 * 8 for e in wl.layer_params) * 2 * 2 + 255) // 256 * 256
    assert store - base == 8 * (4096 * ldy * 2 + wl.s * 4096 * 1024 * 2 + 4096 * 1024 * 4 - grads_saved - slot)


def test_step_cfg_layout_matches_header():
    from paper_2205_00119_b200._lib import StepCfg, StepStats
    text = open(os.path.join(ROOT, "include", "mics.h")).read()
    body = text[text.index("typedef struct {\n  int p, s, nlayers;"):text.index("} mics_step_cfg;")]
    names = re.findall(r"\b(\w+)\s*(?:,|;)", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    assert [f[0] for f in StepCfg._fields_] == names
    assert StepStats._fields_[-4:] == [("compute_flops", C.c_double), ("gemm_launches", C.c_uint64),
                                      ("gather_slots", C.c_uint64), ("gather_slot_bytes", C.c_uint64)]


def test_trace_report_parses(tmp_path):
    rows = ["0,step,-1,-1,0,0", "0,gather,0,0,0.0,0.05", "0,fwd,0,0,0.06,0.20", "0,gather,0,1,0.07,0.10", "0,fwd,0,1,0.25,0.40",
            "0,gather,0,1,0.41,0.45", "0,bwd,0,1,0.46,0.70", "0,gather,0,0,0.50,0.55", "0,bwd,0,0,0.71,0.90",
            "0,rs,0,-1,0.91,1.20", "0,boundary,1,-1,1.21,1.50"]
    p = tmp_path / "t.csv"
    p.write_text("\n".join(rows) + "\n")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "trace_report.py"), str(p), "0"],
                         capture_output=True, text=True, check=True).stdout
    assert "steps traced 1;" in out and "GEMM-stream gaps" in out and "boundary" in out
