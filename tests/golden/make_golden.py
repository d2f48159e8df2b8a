"""Generate the golden vectors that pin the CPU oracle (and, through it, the GPU path).

Everything here is produced by the UNMODIFIED reference hot path compiled from
/root/reference (oracle/_ref/libsdpsim_ref.so via oracle/ref_shim.cpp), using the
reference tests' own generators (std::mt19937 + libstdc++ distributions) and seeds:

  test_collectives.cpp:43-234     KATs, hierarchical sweep, corrupt layout, traffic
  test_sync_schedule.cpp:32-150   int64 sweep, float case, events, state machine
  test_topology.cpp:7-259         layouts, shape table, min feasible partition
  acceptance_main.cpp:50-152      criteria 1 and 2 (digests)

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py
Outputs: tests/golden/reference.npz (arrays) + tests/golden/reference_digests.json.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import RefLib, build_ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def traffic_list(t: dict) -> list:
    return sorted([a, b, c] for (a, b), c in t.items())


def main():
    if not build_ref():
        raise SystemExit("reference not available: cannot generate golden vectors")
    ref = RefLib()
    arr: dict[str, np.ndarray] = {}
    dig: dict[str, object] = {}

    # ---- generators (seeds the reference tests use)
    for seed in (0, 1, 3, 5, 7, 11):
        arr[f"gen/shards/{seed}"] = ref.random_shards(4, 1024, seed).ravel()
    for seed in (1, 42, 2205, 1234):
        arr[f"gen/i64/{seed}"] = ref.random_i64(4096, -1000, 1000, seed)
        arr[f"gen/i64_5/{seed}"] = ref.random_i64(512, -5, 5, seed)
        arr[f"gen/f32/{seed}"] = ref.random_f32(4096, -1.0, 1.0, seed)
    arr["gen/f32/9"] = ref.random_f32(128, -1.0, 1.0, 9)

    # ---- collectives KATs (test_collectives.cpp)
    ag, t = ref.all_gather(np.array([[1], [2], [3]], np.uint8))
    arr["kat/ag_123"] = ag
    sh = ref.random_shards(4, 16, 7)
    _, t = ref.all_gather(sh, ranks=[4, 5, 6, 7])
    dig["kat/ag_traffic_4567"] = traffic_list(t)
    rs, t = ref.reduce_scatter(np.array([[1, 2, 3, 4], [10, 20, 30, 40]], np.int64), "i64")
    arr["kat/rs_i64"] = rs
    arb = np.array([[r, 10 * r, -r, 0] for r in range(4)], np.int64)
    arr["kat/ar_i64"] = ref.all_reduce(arb, "i64")[0]
    # float RS p=8 on 16 floats from mt19937(9) U(-1,1) (test_collectives.cpp:194-206)
    f = ref.random_f32(8 * 16, -1.0, 1.0, 9).reshape(8, 16)
    arr["kat/rs_f32_in"] = f
    arr["kat/rs_f32_out"] = ref.reduce_scatter(f, "f32")[0]
    arr["kat/rs_f32_out_t8"] = ref.reduce_scatter(f, "f32", threads=8)[0]
    # errors: SizeMismatch / TypeMismatch codes
    for name, bufs in (("err/ragged", np.zeros((2, 12), np.uint8)),):
        try:
            ref.reduce_scatter(bufs, "i64")
            dig[name] = 0
        except Exception as e:  # noqa: BLE001
            dig[name] = e.code

    # ---- hierarchical sweep (test_collectives.cpp:98-121): digests of outputs + traffic
    hs = {}
    for k in (1, 2, 4, 8):
        for p in range(k, 65, k):
            for seed in (0, 1):
                for chunk in (1, 7):
                    shards = ref.random_shards(p, chunk, seed)
                    out, tr = ref.hier_all_gather(shards, p, k)
                    flat, _ = ref.all_gather(shards)
                    assert np.array_equal(out, flat)
                    hs[f"{k}/{p}/{seed}/{chunk}"] = [digest(out), sum(tr.values()),
                                                     sum(c for (a, b), c in tr.items() if a // k != b // k)]
    dig["hier/sweep"] = hs
    # multi-group (:123-140)
    shards = ref.random_shards(8, 9, 3)
    arr["hier/multi_in"] = shards
    arr["hier/multi_out"] = ref.hier_all_gather(shards, 4, 2)[0]
    # corrupt layouts (:142-158) and probe p=8,k=4
    arr["hier/corrupt_p4k2"] = ref.hier_all_gather(np.arange(4, dtype=np.uint8).reshape(4, 1), 4, 2, True)[0]
    arr["hier/corrupt_p8k4"] = ref.hier_all_gather(np.arange(8, dtype=np.uint8).reshape(8, 1), 8, 4, True)[0]
    arr["hier/corrupt_n8p4k2_c3"] = ref.hier_all_gather(ref.random_shards(8, 3, 5), 4, 2, True)[0]
    # inter-node traffic (:160-177)
    out, tr = ref.hier_all_gather(ref.random_shards(16, 32, 11), 16, 4)
    dig["hier/traffic_p16k4c32"] = traffic_list(tr)
    # acceptance criterion 1 (acceptance_main.cpp:50-88), digests only
    c1 = {}
    for k in (1, 2, 4, 8):
        for p in range(k, 65, k):
            for seed in range(5):
                for chunk in (1, 7, 1024):
                    shards = ref.random_shards(p, chunk, seed * 977 + p)
                    out, _ = ref.hier_all_gather(shards, p, k)
                    c1[f"{k}/{p}/{seed}/{chunk}"] = digest(out)
    dig["acceptance1"] = c1

    # ---- sync schedule (test_sync_schedule.cpp)
    def grads_i64(s, n, length, lo, hi, seed):
        return ref.random_i64(s * n * length, lo, hi, seed).reshape(s, n, length)

    def grads_f32(s, n, length, seed):
        return ref.random_f32(s * n * length, -1.0, 1.0, seed).reshape(s, n, length)

    for n in (2, 4, 8, 16):
        for p in range(1, n + 1):
            if n % p:
                continue
            for s in (1, 2, 4):
                g = grads_i64(s, n, 13, -1000, 1000, n * 100 + p * 10 + s)
                for mode in ("two_hop", "alternative", "global_sync"):
                    arr[f"sched/i64/{n}/{p}/{s}/{mode}"] = ref.schedule(mode, g, n, p, "i64")[0]
                # acceptance criterion 2 (acceptance_main.cpp:93-152): seed n*1000+p*10+s, i64 then f32
                # (each case draws its own generator; sync_case:97)
                ga = grads_i64(s, n, 13, -1000, 1000, n * 1000 + p * 10 + s)
                arr[f"acc2/i64/{n}/{p}/{s}"] = ref.schedule("two_hop", ga, n, p, "i64")[0]
                gf = grads_f32(s, n, 13, n * 1000 + p * 10 + s)
                for mode in ("two_hop", "alternative", "global_sync"):
                    arr[f"acc2/f32/{n}/{p}/{s}/{mode}"] = ref.schedule(mode, gf, n, p, "f32")[0]
    g = grads_f32(3, 8, 21, 42)
    for mode in ("two_hop", "alternative", "global_sync"):
        arr[f"sched/f32/8/4/3/{mode}"] = ref.schedule(mode, g, 8, 4, "f32")[0]
    # events (:91-115)
    g = grads_i64(2, 8, 16, -5, 5, 1)
    out, ev, tr = ref.schedule("two_hop", g, 8, 4, "i64")
    arr["sched/events_two_hop"] = ev
    dig["sched/events_traffic"] = traffic_list(tr)
    out, ev, tr = ref.schedule("alternative", g, 8, 4, "i64")
    arr["sched/events_alt"] = ev
    # C1-shaped float probe: n=8, p=2, s=4, len=1001, seed 2205
    g = grads_f32(4, 8, 1001, 2205)
    arr["sched/c1probe/two_hop"] = ref.schedule("two_hop", g, 8, 2, "f32")[0]
    arr["sched/c1probe/alternative"] = ref.schedule("alternative", g, 8, 2, "f32")[0]
    # BASELINE config C1 at full size (4 x 1,049,600 = 4,198,400 params as
    # one gradient segment, n=8, p=2, s=4, fp32 U(-1,1) from mt19937(2205)): per-rank
    # digests of the shards after the reference's two_hop and alternative schedules
    # (8 engine threads; the reference pins results for any thread count)
    g = grads_f32(4, 8, 4_198_400, 2205)
    for mode in ("two_hop", "alternative"):
        out = ref.schedule(mode, g, 8, 2, "f32", threads=8)[0]
        dig[f"cfg/c1_full/{mode}"] = [digest(o) for o in out]
        arr[f"cfg/c1_full/{mode}_every_9973"] = out[:, ::9973].copy()
    del g
    # f64 case
    g64 = grads_f32(2, 4, 10, 77).astype(np.float64)
    arr["sched/f64/two_hop"] = ref.schedule("two_hop", g64, 4, 2, "f64")[0]
    # state machine (:117-132)
    arr["sched/state_machine"] = ref.state_machine(4, 2, 2, 8, "bmbmmbm")

    # ---- topology (test_topology.cpp)
    for n in (4, 8, 12, 16, 24):
        for p in range(1, n + 1):
            if n % p == 0:
                part, repl = ref.build_group_layout(n, p)
                arr[f"topo/layout/{n}/{p}/part"] = part
                arr[f"topo/layout/{n}/{p}/repl"] = repl
    bad = {}
    for n, p in ((8, 3), (8, 0), (4, 8), (0, 1), (6, 4)):
        try:
            ref.build_group_layout(n, p)
            bad[f"{n}/{p}"] = 0
        except Exception as e:  # noqa: BLE001
            bad[f"{n}/{p}"] = e.code
    dig["topo/bad_layouts"] = bad
    dig["topo/shape_ok"] = {f"{p}/{k}": ref.partition_shape_ok(p, k) for p in range(0, 17) for k in range(0, 9)}
    mf = {}
    for states in (1 << 30, 160 << 30, 10 << 40, 161_202_626_560):
        for nodes, k, mem in ((8, 8, 32 << 30), (1, 8, 192_000_000_000), (2, 4, 180 << 30)):
            for gran in (0, 1):
                try:
                    mf[f"{states}/{nodes}/{k}/{mem}/{gran}"] = ref.min_feasible_partition(states, nodes, k, mem, gran)
                except Exception as e:  # noqa: BLE001
                    mf[f"{states}/{nodes}/{k}/{mem}/{gran}"] = -e.code
    dig["topo/min_feasible"] = mf

    np.savez_compressed(os.path.join(OUT, "reference.npz"), **arr)
    with open(os.path.join(OUT, "reference_digests.json"), "w") as fh:
        json.dump(dig, fh, indent=0, sort_keys=True)
    print(f"wrote {len(arr)} arrays, {len(dig)} digest groups")


if __name__ == "__main__":
    main()
