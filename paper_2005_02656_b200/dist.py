"""Multi-GPU plumbing: one process per GPU, torch.distributed for bootstrap only.

The data path (halo exchanges, migration, dt / bbox / histogram allreduces) runs
inside libsph over its own NCCL communicator; this module only (1) initialises
the process group, (2) broadcasts rank 0's NCCL unique id, (3) gathers per-rank
results for checks.  Launch: ``python -m torch.distributed.run --nproc-per-node N
--master-addr 127.0.0.1 ...`` (RANK / LOCAL_RANK / WORLD_SIZE from the env).
"""
from __future__ import annotations

import os

import numpy as np


def env() -> tuple[int, int, int]:
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str = "nccl") -> tuple[int, int, int]:
    import torch
    import torch.distributed as dist
    world, rank, local = env()
    if backend == "nccl":
        torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group(backend, init_method="env://")
    return world, rank, local


def share_unique_id(rank: int, world: int, device: str = "cuda") -> bytes | None:
    """Rank 0 creates the NCCL id through the C ABI; everyone receives the same bytes."""
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist

    from . import sph
    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(sph.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())


def gather_by_id(state: dict, world: int, fields) -> dict | None:
    """Concatenate every rank's owned particles on rank 0, ordered by global id."""
    import torch.distributed as dist
    local = {k: np.asarray(state[k]) for k in ("id",) + tuple(fields)}
    if world <= 1:
        parts = [local]
    else:
        parts = [None] * world
        dist.all_gather_object(parts, local)
    if dist.is_initialized() and dist.get_rank() != 0:
        return None
    out = {k: np.concatenate([p[k] for p in parts]) for k in local}
    order = np.argsort(out["id"], kind="stable")
    return {k: v[order] for k, v in out.items()}


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
