"""Multi-GPU plumbing: one process per GPU (torchrun), NCCL communicator for the
library's own collectives, and the shard arithmetic shared with the C ABI.

Full spectrum: Z is column-sharded, rank r owns columns [n*r//g, n*(r+1)//g)
(csrc/ipt_internal.cuh Ctx::shard); Delta and d are replicated; per iteration one
all-reduce of {sum|F-Z|^2, sum|Z|^2, sum|F|^2} (+ max|F-Z|). Single pair (CSR):
rows are sharded in equal chunks ceil(n/g) (csrc/ipt_single.cu), z is
all-gathered in place after every step.
"""
from __future__ import annotations

import os

from .ipt import Context, nccl_unique_id


def column_shard(n: int, rank: int, nranks: int) -> tuple[int, int]:
    return n * rank // nranks, n * (rank + 1) // nranks


def row_chunk(n: int, rank: int, nranks: int) -> tuple[int, int]:
    chunk = -(-n // nranks)
    return min(n, rank * chunk), min(n, (rank + 1) * chunk)


def init_context_from_env() -> Context:
    """Context on LOCAL_RANK's GPU; with WORLD_SIZE > 1 a NCCL communicator whose
    unique id is broadcast over torch.distributed (the process group is plumbing only)."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    ctx = Context(local)
    if world > 1:
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.init_comm(obj[0], rank, world)
    return ctx
