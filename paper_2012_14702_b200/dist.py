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

import threading
from typing import Callable, Sequence

from .ipt import Context, LocalGroup, nccl_unique_id


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


def local_contexts(nranks: int, devices: Sequence[int] = (0,)) -> list[Context]:
    """nranks contexts of this process joined in one in-process communicator group
    (ipt_ctx_init_local_comm); rank r runs on devices[r % len(devices)]. With one
    device this drives the library's multi-rank code (sharded upload, per-iteration
    all-reduce, fused peer-store all-gather, gathers) on a single GPU."""
    group = LocalGroup(nranks)
    ctxs = []
    for r in range(nranks):
        c = Context(devices[r % len(devices)])
        c.init_local_comm(group, r)
        ctxs.append(c)
    return ctxs


def run_ranks(fn: Callable[[Context], object], ctxs: Sequence[Context]) -> list:
    """fn(ctx) on one host thread per rank (ctypes releases the GIL inside the library);
    returns the per-rank results, re-raising the first rank's exception."""
    out: list = [None] * len(ctxs)
    err: list = [None] * len(ctxs)

    def body(r):
        try:
            out[r] = fn(ctxs[r])
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(len(ctxs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out
