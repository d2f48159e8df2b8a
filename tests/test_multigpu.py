"""Multi-GPU / multi-process tests.

* CPU (gloo, world_size 2): the host-side planning of the multi-process layout
  (node-major rank placement, barrier peer sets, IPC-handle exchange protocol).
* GPU (>= 2 GPUs): tests/mp_worker.py under torchrun — every collective across
  processes over NVLink peer memory, bit-exact against the oracle.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2205_00119_b200 import dist as mdist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = mdist.exchange(bytes([rank]) * 64, world)  # the IPC-handle exchange protocol
        assert got == [bytes([r]) * 64 for r in range(world)]
        local = mdist.plan_local_ranks(8, world, rank)
        allr = mdist.exchange(local, world)
        assert sorted(sum(allr, [])) == list(range(8))
        peers = mdist.barrier_peers(8, world, 2, rank)
        peer_sets = mdist.exchange(peers, world)
        # barrier peer relation must be symmetric, or pairwise flag counters drift
        for kind in ("partition", "replication"):
            for a in range(world):
                for b in peer_sets[a][kind]:
                    assert a in peer_sets[b][kind], (kind, a, b)
        q.put((rank, "ok", peers))
    except Exception as e:  # noqa: BLE001
        q.put((rank, f"fail: {e!r}", None))
    finally:
        dist.destroy_process_group()


def test_multiprocess_host_plumbing_gloo():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29400 + os.getpid() % 500
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == ["ok", "ok"], res
    # n=8 over 2 processes, p=2: partition groups are process-local, replication groups cross
    assert res[0][2] == {"partition": [], "replication": [1]}


def test_barrier_peers_layouts():
    sys.path.insert(0, ROOT)
    from paper_2205_00119_b200.dist import barrier_peers, plan_local_ranks
    assert plan_local_ranks(8, 4, 1) == [2, 3]
    # n=8 on 8 GPUs, p=4: partition peers are the 3 other GPUs of the group
    assert barrier_peers(8, 8, 4, 5) == {"partition": [4, 6, 7], "replication": [1]}
    assert barrier_peers(8, 2, 8, 0) == {"partition": [1], "replication": []}
    with pytest.raises(ValueError):
        plan_local_ranks(8, 3, 0)


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("world", [2, 4])
def test_collectives_across_gpus(world):
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, MICS_TEST_RANKS="8")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world), os.path.join(ROOT, "tests", "mp_worker.py")]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert out.stdout.count("ok (") == world
