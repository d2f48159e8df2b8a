"""Multi-process plumbing: one process per GPU (torchrun), CUDA IPC handles of
every process's arena exchanged over ``torch.distributed``.  torch is used only
for the rendezvous / handle exchange (and by bench.py for the NCCL comparator);
all data movement is libmics's own kernels over NVLink peer memory."""
from __future__ import annotations

import os

from .engine import Engine


def env_world():
    """(rank, world, local_rank) from torchrun's environment (1-process defaults)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def exchange(obj, world: int, group=None):
    """all_gather_object over `group` (default: the default process group)."""
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, obj, group=group)
    return out


def connect(engine: Engine, group=None) -> None:
    """Export this process's arena handle, import everybody's (world order)."""
    if engine.world == 1:
        return
    handles = exchange(engine.export_handle(), engine.world, group)
    engine.import_handles(handles)


def init_engine(n_ranks: int, arena_bytes: int, backend: str = "gloo") -> Engine:
    """Create the engine for this process (device = LOCAL_RANK) and connect it."""
    rank, world, local = env_world()
    if world > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group(backend=backend)
    engine = Engine(n_ranks=n_ranks, world=world, world_rank=rank, device=local, arena_bytes=arena_bytes)
    connect(engine)
    return engine


def plan_local_ranks(n_ranks: int, world: int, rank: int) -> list:
    """Node-major placement used by libmics (include/mics.h): n/world contiguous ranks per process."""
    if n_ranks % world:
        raise ValueError("world must divide n_ranks")
    per = n_ranks // world
    return list(range(rank * per, (rank + 1) * per))


def barrier_peers(n_ranks: int, world: int, p: int, rank: int) -> dict:
    """Processes each process exchanges flag barriers with, per collective kind
    (host restatement of mics_ctx::peer_mask, for CPU tests and planning)."""
    per = n_ranks // world
    mine = set(plan_local_ranks(n_ranks, world, rank))

    def peers(groups):
        out = set()
        for g in groups:
            if mine & set(g):
                out |= {r // per for r in g}
        out.discard(rank)
        return sorted(out)

    part = [list(range(g * p, (g + 1) * p)) for g in range(n_ranks // p)]
    repl = [list(range(j, n_ranks, p)) for j in range(p)]
    return {"partition": peers(part), "replication": peers(repl)}
