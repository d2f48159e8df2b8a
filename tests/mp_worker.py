"""Multi-process worker for tests/test_multigpu.py (one process per GPU, torchrun).

Every process builds the same job (n virtual ranks over `world` GPUs, node-major),
maps the peers' arenas through CUDA IPC and runs the collectives across GPUs over
NVLink; each process checks the ranks it hosts against the CPU oracle.
Exit status 0 = every check passed.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2205_00119_b200 import dist as mdist
    from paper_2205_00119_b200.collectives import (all_gather_device, all_reduce_device,
                                                   hierarchical_all_gather_device, reduce_scatter_device)
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.sync_schedule import AdamConfig, SyncStates, make_adam
    from paper_2205_00119_b200.topology import build_group_layout

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    n = int(os.environ.get("MICS_TEST_RANKS", 8))
    ora = Oracle()
    eng = Engine(n_ranks=n, world=world, world_rank=rank, device=local, arena_bytes=1 << 30)
    mdist.connect(eng)
    mine = eng.local_ranks
    fails = []

    def expect(cond, what):
        if not cond:
            fails.append(what)

    # ---- partition-group all-gather, p in {2, 4, n}: groups span GPUs when p > n/world
    for p in (2, 4, n):
        chunk = (1 << 20) + 48
        src, dst = eng.alloc(chunk), eng.alloc(p * chunk)
        shards = ora.random_shards(n, chunk, 100 + p)
        for r in mine:
            eng.h2d(src, r, shards[r])
        eng.barrier()
        for g in range(n // p):
            ranks = list(range(g * p, (g + 1) * p))
            all_gather_device(eng, ranks, [eng.ptr(src, r) for r in ranks], chunk,
                              [eng.ptr(dst, r) if r in mine else 0 for r in ranks])
        eng.synchronize()
        for r in mine:
            g = r // p
            expect(np.array_equal(eng.d2h(dst, r, p * chunk, "u8"),
                                  shards[g * p:(g + 1) * p].ravel()), f"all_gather p={p} r={r}")

    # ---- reduce-scatter f32 across GPUs, bit-exact
    for p in (2, 4, n):
        chunk = 300_007
        src, dst = eng.alloc(4 * p * chunk), eng.alloc(4 * chunk)
        bufs = np.stack([ora.random_f32(p * chunk, -1, 1, 7 * r + p) for r in range(n)])
        for r in mine:
            eng.h2d(src, r, bufs[r])
        eng.barrier()
        for g in range(n // p):
            ranks = list(range(g * p, (g + 1) * p))
            reduce_scatter_device(eng, ranks, [eng.ptr(src, r) for r in ranks], p * chunk,
                                  [eng.ptr(dst, r) if r in mine else 0 for r in ranks], "f32")
        eng.synchronize()
        for r in mine:
            g = r // p
            want = ora.reduce_scatter(bufs[g * p:(g + 1) * p], "f32")[r % p]
            expect(np.array_equal(eng.d2h(dst, r, chunk).view(np.uint32), want.view(np.uint32)), f"rs p={p} r={r}")

    # ---- all-reduce in replication groups (stride p)
    p = 2
    elems = 4 * 65_537
    buf = eng.alloc(4 * elems)
    bufs = np.stack([ora.random_f32(elems, -1, 1, 900 + r) for r in range(n)])
    for r in mine:
        eng.h2d(buf, r, bufs[r])
    eng.barrier()
    for j in range(p):
        ranks = list(range(j, n, p))
        all_reduce_device(eng, ranks, [eng.ptr(buf, r) for r in ranks], elems, "f32")
    eng.synchronize()
    for r in mine:
        ranks = list(range(r % p, n, p))
        want = ora.all_reduce(bufs[ranks], "f32")[0]
        expect(np.array_equal(eng.d2h(buf, r, elems).view(np.uint32), want.view(np.uint32)), f"all_reduce r={r}")

    # ---- hierarchical all-gather (k ranks per virtual node), incl. the corrupt hook
    for p, k, corrupt in ((n, n // 2, False), (4, 2, False), (n, 2, True)):
        chunk = 65_536 + 16
        src, dst = eng.alloc(chunk), eng.alloc(p * chunk)
        shards = ora.random_shards(n, chunk, 55 + p + k)
        for r in mine:
            eng.h2d(src, r, shards[r])
        eng.barrier()
        hierarchical_all_gather_device(eng, p, k, [eng.ptr(src, r) for r in range(n)], chunk,
                                       [eng.ptr(dst, r) for r in range(n)], corrupt)
        eng.synchronize()
        want = ora.hier_all_gather(shards, p, k, corrupt)
        for r in mine:
            expect(np.array_equal(eng.d2h(dst, r, p * chunk, "u8"), want[r]),
                   f"hier p={p} k={k} corrupt={corrupt} r={r}")

    # ---- 2-hop schedule + fused Adam across GPUs
    for p in (2, 4):
        s, length = 3, 200_003
        lay = build_group_layout(n, p)
        st = SyncStates(eng, lay, [length], s, "f32")
        grads = ora.random_f32(s * n * length, -1, 1, 31 + p).reshape(s, n, length)
        gb = eng.alloc(4 * st.grad_elems)
        for t in range(s):
            for r in mine:
                eng.h2d(gb, r, grads[t, r])
            eng.barrier()
            st.micro_step_device(gb)
            eng.synchronize()
        c = st.shard_elems
        pb, mb, vb = (eng.alloc(4 * c) for _ in range(3))
        p0 = ora.random_f32(c, -1, 1, 3)
        for r in mine:
            eng.h2d(pb, r, p0)
            eng.memset(mb, r, 4 * c)
            eng.memset(vb, r, 4 * c)
        eng.barrier()
        st.boundary(make_adam(st, AdamConfig(lr=1e-3, grad_scale=0.5, write_grad=True), pb, mb, vb))
        eng.synchronize()
        want, _, _ = ora.two_hop(grads, n, p, "f32")
        for r in mine:
            expect(np.array_equal(st.shard(r).view(np.uint32), want[r].view(np.uint32)), f"two_hop p={p} r={r}")
            wp, _, _, _ = ora.adam(p0, np.zeros(c), np.zeros(c), want[r], 1e-3, 0.9, 0.999, 1e-8, 0, 1, 0.5)
            expect(np.array_equal(eng.d2h(pb, r, c).view(np.uint32), wp.view(np.uint32)), f"adam p={p} r={r}")
        st.close()

    eng.synchronize()
    eng.close()

    # ---- the MiCS step driver across processes: 2-hop (flat + hierarchical) and the
    # alternative schedule, bit-exact against the CPU restatement of the step
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    from test_gpu_step import expected_step
    for p, k, alt, gdt in ((2, 0, False, "f32"), (4, 2, False, "bf16"), (4, 0, True, "f32"), (8, 0, False, "f32"),
                           (8, 4, False, "bf16")):
        e2 = Engine(n_ranks=n, world=world, world_rank=rank, device=local, arena_bytes=256 << 20)
        mdist.connect(e2)
        wl = Workload("mp", [20_000, 4_099, 65_536], p=p, s=2, grad_dtype=gdt, hier_k=k)
        opts = StepOptions(resident_grads=not alt, alternative=alt, seed=91, lr=1e-3)
        step = MicsStep(e2, wl, opts)
        info, segs = step.sync_info()
        bufs = step.buffers()
        step.run(1)
        e2.synchronize()
        want, _ = expected_step(ora, n, p, 2, segs, gdt, 91, alt, opts)
        for r in e2.local_ranks:
            got = e2.d2h(bufs["master"], r, info.shard_elems)
            expect(np.array_equal(got.view(np.uint32), want[r][0].view(np.uint32)),
                   f"step p={p} k={k} alt={alt} {gdt} r={r}")
        step.close()
        e2.close()

    # ---- merged hierarchical launches (flags across processes; node peers on other GPUs
    # for p=8, k=4) vs one k_hier launch per visit, over 3 steps: same bits
    for p, k in ((4, 2), (8, 4)):
        res = {}
        for merge in ("1", "0"):
            os.environ["MICS_HIER_MERGE"] = merge
            e7 = Engine(n_ranks=n, world=world, world_rank=rank, device=local, arena_bytes=256 << 20)
            mdist.connect(e7)
            step = MicsStep(e7, Workload("hm", [70_000, 12_345, 40_000, 9_999, 33_333], p=p, s=2, hier_k=k),
                            StepOptions(seed=5))
            step.run(3)
            e7.synchronize()
            S = step.sync_info()[0].shard_elems
            b = step.buffers()
            half, slots = step.stats().gather_slot_bytes, step.stats().gather_slots
            segs = step.sync_info()[1]
            res[merge] = [e7.d2h(b["master"], r, S) for r in e7.local_ranks] + \
                         [e7.d2h(b["gathered"], r, p * segs[l][1], "bf16", off=(l % slots) * half)
                          for r in e7.local_ranks for l in range(3)]
            step.close()
            e7.close()
        os.environ.pop("MICS_HIER_MERGE")
        for x, y in zip(res["0"], res["1"]):
            expect(np.array_equal(x.view(np.uint16), y.view(np.uint16)), f"hier merged != per-visit (p={p}, k={k})")

    # ---- full-size C3 step across processes: sampled elements bit-exact (test_gpu_fullsize)
    from test_gpu_fullsize import check_sampled
    import bench
    from paper_2205_00119_b200.step import workloads
    wl3 = workloads()["C3"]
    opts3 = StepOptions(seed=2205, lr=1e-4)
    e6 = Engine(n_ranks=n, world=world, world_rank=rank, device=local,
                arena_bytes=bench.arena_bytes(wl3, n // world, True, n))
    mdist.connect(e6)
    step = MicsStep(e6, wl3, opts3)
    step.run(1)
    e6.synchronize()
    try:
        check_sampled(ora, e6, step, wl3, opts3, e6.local_ranks, nsamples=150, seed=rank)
    except AssertionError as ex:
        expect(False, f"full-size C3 sampled check: {ex}")
    # every element of every local rank's master and bf16 shard (the K9 boundary across
    # processes) against the oracle's whole-shard step
    info3, segs3 = step.sync_info()
    S3 = info3.shard_elems
    for j in sorted({r % wl3.p for r in e6.local_ranks}):
        want, _, _, want_bf = ora.step1_shard(opts3.seed, wl3.n, wl3.p, wl3.s, j, segs3, S3, opts3.lr,
                                              threads=max(1, (os.cpu_count() or 4) // world))
        for r in e6.local_ranks:
            if r % wl3.p != j:
                continue
            got = e6.d2h(step.buffers()["master"], r, S3)
            nbad = int(np.count_nonzero(got.view(np.uint32) != want.view(np.uint32)))
            expect(nbad == 0, f"full-size C3 master of rank {r}: {nbad} elements differ")
            expect(np.array_equal(e6.d2h(step.buffers()["param_bf16"], r, S3, "bf16"), want_bf),
                   f"full-size C3 bf16 of rank {r}")
    step.close()
    e6.close()

    # ---- overlapped tail (auto-on for multi-process jobs) vs in order; p=4 spans GPUs at world 4
    for pt in (2, 4):
        res = {}
        for tail in ("0", "1", "1f"):
            os.environ["MICS_TAIL_OVERLAP"] = tail[0]
            os.environ["MICS_TAIL_FUSED"] = "1" if tail == "1f" else "0"
            e5 = Engine(n_ranks=n, world=world, world_rank=rank, device=local, arena_bytes=256 << 20)
            mdist.connect(e5)
            step = MicsStep(e5, Workload("tail", [1_500_000, 70_000, 12_345, 700_000, 40_000, 9_999, 33_333], p=pt, s=3),
                            StepOptions(seed=5))
            step.run(2)
            step.profile()
            step.run(1)
            e5.synchronize()
            S = step.sync_info()[0].shard_elems
            res[tail] = [e5.d2h(step.buffers()["master"], r, S) for r in e5.local_ranks]
            step.close()
            e5.close()
        os.environ.pop("MICS_TAIL_OVERLAP")
        os.environ.pop("MICS_TAIL_FUSED")
        for t in ("1", "1f"):
            for x, y in zip(res["0"], res[t]):
                expect(np.array_equal(x.view(np.uint32), y.view(np.uint32)),
                       f"overlapped tail ({t}) != in-order (p={pt})")

    # ---- the step with compute across processes (gathers / GEMMs / sync on three
    # streams, hierarchical gathers on barrier channel 1): GEMM gradients within
    # tolerance of fp32, the sync + Adam bit-exact on the gradients the GEMMs produced
    from test_gpu_step_compute import bf16_bits_to_f32, f32_to_bf16_bits, layer_weights, reduce_and_adam
    for p, k, gdt in ((2, 0, "f32"), (4, 2, "bf16"), (8, 0, "f32")):
        e4 = Engine(n_ranks=n, world=world, world_rank=rank, device=local, arena_bytes=256 << 20)
        mdist.connect(e4)
        h = 64
        wl = Workload("mpc", [h * 40, h * 37, h * 56], p=p, s=2, grad_dtype=gdt, hier_k=k, hidden=h, seq_len=16)
        opts = StepOptions(seed=91, lr=1e-3, compute=True)
        step = MicsStep(e4, wl, opts)
        info, segs = step.sync_info()
        S, G, T = info.shard_elems, info.grad_elems, wl.tokens
        b = step.buffers()
        gsz = 2 if gdt == "bf16" else 4
        for stepno in (1, 2):
            pb_loc = {r: e4.d2h(b["param_bf16"], r, S, "bf16") for r in e4.local_ranks}
            init_loc = {r: (e4.d2h(b["master"], r, S), e4.d2h(b["exp_avg"], r, S), e4.d2h(b["exp_avg_sq"], r, S))
                        for r in e4.local_ranks}
            step.run(1)
            e4.synchronize()
            g_loc = {}
            for r in e4.local_ranks:
                gr = np.zeros((2, G), np.float32)
                for t in range(2):
                    raw = e4.d2h(b["grads"], r, G, gdt, off=t * G * gsz)
                    gr[t] = bf16_bits_to_f32(raw) if gdt == "bf16" else raw
                g_loc[r] = gr
            allg = [None] * world
            dist.all_gather_object(allg, (pb_loc, g_loc, init_loc))
            pb, grads, init = {}, np.zeros((2, n, G), np.float32), {}
            for d_pb, d_g, d_init in allg:
                pb.update(d_pb)
                init.update(d_init)
                for r, gr in d_g.items():
                    grads[:, r] = gr
            for r in e4.local_ranks:  # GEMM gradients vs fp32 (tolerance)
                g = r // p
                Ws = layer_weights(pb, segs, h, p, lambda i: g * p + i)
                for t in range(2):
                    X = bf16_bits_to_f32(ora.gen_bf16(91 ^ 0xA11CE, r, t, 254, 0, T * h)).reshape(T, h)
                    for (ln, c, so, go), W in zip(segs, Ws):
                        Y = bf16_bits_to_f32(f32_to_bf16_bits(X @ W.T))
                        dW = (Y.T @ X).ravel()
                        bound = 2e-2 * (np.abs(Y).T @ np.abs(X)).ravel() + 1e-5 + (np.abs(dW) * 2.0 ** -8 if gdt == "bf16" else 0)
                        expect(bool(np.all(np.abs(grads[t, r, go:go + ln] - dW) <= bound)),
                               f"compute step p={p} k={k} step={stepno} r={r} t={t}: dW")
            want = reduce_and_adam(ora, n, p, 2, segs, grads, [init[r] for r in range(n)], opts, step=stepno)
            for r in e4.local_ranks:
                expect(np.array_equal(e4.d2h(b["master"], r, S).view(np.uint32), want[r][0].view(np.uint32)),
                       f"compute step p={p} k={k} step={stepno} r={r}: master")
        step.close()
        e4.close()

    dist.barrier()
    if fails:
        print(f"[rank {rank}] FAILED: {fails}", flush=True)
        sys.exit(1)
    print(f"[rank {rank}] ok ({len(mine)} local ranks)", flush=True)


if __name__ == "__main__":
    main()
