"""Can two processes form a NCCL communicator on ONE GPU (to run the library's NCCL backend
for real on this one-GPU pool)? torchrun --nproc-per-node 2, both on cuda:0."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
ctx = ipt.Context(0)
obj = [ipt.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
try:
    ctx.init_comm(obj[0], rank, world)
    print(f"rank {rank}: NCCL communicator on one GPU OK ({ctx.comm_kind})", flush=True)
    p = synth.dense_uniform(512, 0.02, 42)
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12), ctx=ctx)
    if rank == 0:
        one = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12), ctx=ipt.Context(0))
        print("bitwise vs one rank:", np.array_equal(r.Z, one.Z), flush=True)
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: {type(e).__name__}: {e}", flush=True)
dist.barrier()
