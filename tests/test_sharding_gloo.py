"""The N>1 host logic on CPU (gloo, world_size 2): column-sharded full-spectrum
iteration and row-sharded single-pair iteration with the same shard arithmetic
and collectives the device path uses, checked against the one-rank run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2012_14702_b200.dist import column_shard, row_chunk


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sharded_full(rank, world, port, n, tol, out_q):
    import oracle
    from paper_2012_14702_b200 import synth

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = oracle.port()
    p = synth.dense_uniform(n, 0.02, 5)
    c0, c1 = column_shard(n, rank, world)
    z = np.zeros((n, c1 - c0), np.complex128)
    z[np.arange(c0, c1), np.arange(c1 - c0)] = 1.0
    it = 0
    for k in range(100):
        f, s = P.full_map_block(p.d, p.delta, c0, z)
        t = torch.tensor(s[:3], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        m = torch.tensor([s[3]], dtype=torch.float64)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        step = np.sqrt(t[0].item()) / np.sqrt(t[1].item())
        z = f
        it = k + 1
        if step <= tol:  # every rank takes the identical decision from the reduced scalars
            break
    lam, r2 = P.full_final_block(p.d, p.delta, c0, z)
    r = torch.tensor([r2], dtype=torch.float64)
    dist.all_reduce(r)
    blocks = [None] * world
    dist.all_gather_object(blocks, (c0, z, lam))
    if rank == 0:
        out_q.put((it, step, float(np.sqrt(r.item())), blocks))
    dist.destroy_process_group()


def test_column_sharded_full_iteration_matches_single_rank():
    import oracle

    n, tol = 96, 1e-13
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_full, args=(r, 2, port, n, tol, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    it, step, res, blocks = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    from paper_2012_14702_b200 import synth

    p = synth.dense_uniform(n, 0.02, 5)
    one = oracle.port().solve_full(p.d, p.delta, tol=tol, sigma=False)
    assert it == one["iterations"]
    z = np.concatenate([b[1] for b in sorted(blocks, key=lambda b: b[0])], axis=1)
    lam = np.concatenate([b[2] for b in sorted(blocks, key=lambda b: b[0])])
    # column independence: each shard reproduces its columns of the one-rank run bit for bit
    assert np.array_equal(z, one["Z"])
    assert np.array_equal(lam, one["eigenvalues"])
    assert res == pytest.approx(one["residual_frobenius"], rel=1e-12)


def _sharded_single(rank, world, port, n, anchor, tol, out_q):
    from paper_2012_14702_b200 import synth

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = synth.csr_ci(n, 8, 0.01, 3)
    r0, r1 = row_chunk(n, rank, world)
    chunk = -(-n // world)
    rp, ci, va = p.delta.row_offsets, p.delta.col_indices, p.delta.values
    d = p.d
    # every rank holds row a (w_a computed locally, no broadcast)
    arow = slice(rp[anchor], rp[anchor + 1])
    z = np.zeros(chunk * world)
    z[anchor] = 1.0
    g = 1.0 / (d - d[anchor])
    for k in range(200):
        wa = float(np.dot(va[arow], z[ci[arow]]))
        fz = np.zeros(chunk * world)
        sums = np.zeros(3)
        for i in range(r0, r1):
            w = float(np.dot(va[rp[i]:rp[i + 1]], z[ci[rp[i]:rp[i + 1]]]))
            f = 1.0 if i == anchor else g[i] * (z[i] * wa - w)
            fz[i] = f
            sums += [(z[i] - f) ** 2, z[i] ** 2, f ** 2]
        t = torch.tensor(fz[r0:r0 + chunk] if r1 - r0 == chunk else np.pad(fz[r0:r1], (0, chunk - (r1 - r0))))
        parts = [torch.zeros(chunk, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, t)
        s = torch.tensor(sums)
        dist.all_reduce(s)
        z = torch.cat(parts).numpy().copy()
        step = np.sqrt(s[0].item()) / np.sqrt(s[1].item())
        if step <= tol:
            break
    if rank == 0:
        out_q.put((k + 1, z[:n]))
    dist.destroy_process_group()


def test_row_sharded_single_pair_matches_single_rank():
    import oracle
    from paper_2012_14702_b200 import synth

    n, anchor, tol = 2000, 3, 1e-12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_single, args=(r, 2, port, n, anchor, tol, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    it, z = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = synth.csr_ci(n, 8, 0.01, 3)
    one = oracle.port().solve_single(p.d, p.delta, anchor, tol=tol)
    assert abs(it - one["iterations"]) <= 1
    assert np.max(np.abs(z - one["z"].real)) <= 1e-14


def test_shard_arithmetic_covers_every_index():
    for n in (1, 7, 1000, 32768, (1 << 21) + 3):
        for g in (1, 2, 3, 4, 8):
            cols = [column_shard(n, r, g) for r in range(g)]
            assert cols[0][0] == 0 and cols[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(cols, cols[1:]))
            rows = [row_chunk(n, r, g) for r in range(g)]
            assert rows[0][0] == 0 and rows[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
