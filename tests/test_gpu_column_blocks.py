"""Column blocks of the full-spectrum problem (the unit one rank iterates under the
column sharding of SURVEY §8e, ipt_full.cu): a block [b, e) run alone on one GPU must
reproduce columns b..e-1 of the whole problem BIT FOR BIT -- every kernel of the map
(K2 pre-pass, DMMA map GEMM / identity-start map, SpMM map, 3M complex map, closing
product) addresses global columns through col0. With convergence ignored the loop
length is fixed, so several iterations compare exactly too; eigenvalues likewise,
and the block residuals add up (in squares) to the whole residual.

What one GPU cannot exercise -- the NCCL all-reduce of the stop scalars and the
gather to rank 0 -- is the host logic covered by tests/test_sharding_gloo.py."""
import ctypes as C

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import _lib, synth
from paper_2012_14702_b200._lib import Stats, check, dptr, i32ptr, i64ptr
from paper_2012_14702_b200.ipt import _params

pytestmark = pytest.mark.gpu


def _run(upload, n, warm, iters, want_block, ncols, product=_lib.PRODUCT_DMMA):
    lib = _lib.load()
    ctx = ipt.default_context()
    h = C.c_void_p()
    check(upload(ctx, C.byref(h)))
    try:
        check(lib.ipt_full_set_product(h, product))
        wr = None if warm is None else np.ascontiguousarray(warm.real)
        wi = None if warm is None or not np.iscomplexobj(warm) else np.ascontiguousarray(warm.imag)
        check(lib.ipt_full_reset(ctx.handle, h, dptr(wr), dptr(wi)))
        prm = _params(ipt.IterationConfig(max_iterations=iters), ignore_convergence=1, want_sigma_min=0,
                      divergence_threshold=1e300)
        st = Stats()
        check(lib.ipt_full_iterate(ctx.handle, h, C.byref(prm), C.byref(st)))
        check(lib.ipt_full_finalize(ctx.handle, h, C.byref(prm), C.byref(st)))
        zr, zi = np.empty((n, ncols)), np.empty((n, ncols))
        lr, li = np.empty(ncols), np.empty(ncols)
        if want_block:
            check(lib.ipt_full_download_block(ctx.handle, h, dptr(zr), dptr(zi), dptr(lr), dptr(li)))
        else:
            check(lib.ipt_full_download(ctx.handle, h, dptr(zr), dptr(zi), dptr(lr), dptr(li)))
        return zr + 1j * zi, lr + 1j * li, st.residual, st.iterations
    finally:
        lib.ipt_full_free(h)


def dense_runs(d, dr, di, warm, iters, blocks, product=_lib.PRODUCT_DMMA):
    lib = _lib.load()
    n = len(d)

    def full(ctx, out):
        return lib.ipt_full_upload(ctx.handle, n, dptr(d), None, dptr(dr), dptr(di), out)

    ref = _run(full, n, warm, iters, False, n, product)
    outs = []
    for b, e in blocks:
        def up(ctx, out, b=b, e=e):
            return lib.ipt_full_upload_columns(ctx.handle, n, dptr(d), None, dptr(dr), dptr(di), b, e, out)
        outs.append(((b, e), _run(up, n, warm, iters, True, e - b, product)))
    return ref, outs


def check_blocks(ref, outs, n):
    z, lam, res, it = ref
    r2 = 0.0
    for (b, e), (zb, lb, rb, itb) in outs:
        assert itb == it
        assert np.array_equal(zb, z[:, b:e]), (b, e, np.max(np.abs(zb - z[:, b:e])))
        assert np.array_equal(lb, lam[b:e])
        r2 += rb * rb
    return r2


BLOCKS = [(0, 350), (350, 700), (123, 457), (699, 700), (0, 700)]


@pytest.mark.parametrize("iters", [1, 4])
def test_real_dense_blocks_from_identity(iters):
    n = 700
    p = synth.dense_uniform(n, 0.3 / np.sqrt(n), 7)
    ref, outs = dense_runs(p.d, np.ascontiguousarray(p.delta), None, None, iters, BLOCKS)
    r2 = check_blocks(ref, outs[:2], n)
    assert np.sqrt(r2) == pytest.approx(ref[2], rel=1e-10)
    check_blocks(ref, outs[2:], n)


def test_real_dense_blocks_from_warm_start():
    n = 700
    p = synth.dense_uniform(n, 0.3 / np.sqrt(n), 8)
    rng = np.random.default_rng(1)
    warm = np.eye(n) + 1e-3 * rng.standard_normal((n, n))
    np.fill_diagonal(warm, 1.0)
    ref, outs = dense_runs(p.d, np.ascontiguousarray(p.delta), None, warm, 3, BLOCKS)
    check_blocks(ref, outs, n)


@pytest.mark.parametrize("iters", [1, 3])
def test_ozaki_blocks(iters):
    """The Ozaki-product map (residues per Z column, exact integer products, one rounding
    per entry) is column-local too: blocks reproduce the whole run bit for bit."""
    n = 700
    p = synth.dense_uniform(n, 0.3 / np.sqrt(n), 9)
    rng = np.random.default_rng(2)
    warm = np.eye(n) + 1e-3 * rng.standard_normal((n, n))
    np.fill_diagonal(warm, 1.0)
    for w in (None, warm):
        ref, outs = dense_runs(p.d, np.ascontiguousarray(p.delta), None, w, iters, BLOCKS, _lib.PRODUCT_OZAKI)
        check_blocks(ref, outs, n)


@pytest.mark.parametrize("product", [_lib.PRODUCT_DMMA, _lib.PRODUCT_OZAKI])
def test_complex_blocks(product):
    n = 300
    rng = np.random.default_rng(2)
    d = np.arange(1.0, n + 1)
    dr = 0.02 * rng.standard_normal((n, n))
    di = 0.02 * rng.standard_normal((n, n))
    np.fill_diagonal(dr, 0)
    np.fill_diagonal(di, 0)
    ref, outs = dense_runs(d, dr, di, None, 3, [(0, 128), (128, 300), (37, 201)], product)
    check_blocks(ref, outs, n)


def test_sparse_blocks():
    lib = _lib.load()
    n = 900
    rng = np.random.default_rng(3)
    rows = np.repeat(np.arange(n), 9)
    cols = rng.integers(0, n, rows.size)
    keep = rows != cols
    key = np.unique(np.minimum(rows[keep], cols[keep]) * n + np.maximum(rows[keep], cols[keep]))
    r, c = key // n, key % n
    v = 0.05 * rng.standard_normal(key.size)
    delta = ipt.CsrMatrix.from_triplets(n, n, np.concatenate([r, c]), np.concatenate([c, r]), np.concatenate([v, v]))
    d = np.arange(n, dtype=float)

    def full(ctx, out):
        return lib.ipt_full_upload_csr(ctx.handle, n, dptr(d), None, i64ptr(delta.row_offsets),
                                       i32ptr(delta.col_indices), dptr(delta.values), None, out)

    ref = _run(full, n, None, 3, False, n)
    outs = []
    for b, e in [(0, 450), (450, 900), (300, 301), (5, 777)]:
        def up(ctx, out, b=b, e=e):
            return lib.ipt_full_upload_csr_columns(ctx.handle, n, dptr(d), i64ptr(delta.row_offsets),
                                                   i32ptr(delta.col_indices), dptr(delta.values), b, e, out)
        outs.append(((b, e), _run(up, n, None, 3, True, e - b)))
    check_blocks(ref, outs, n)


def test_bad_blocks_rejected():
    lib = _lib.load()
    ctx = ipt.default_context()
    n = 10
    d = np.arange(n, dtype=float)
    delta = np.zeros((n, n))
    h = C.c_void_p()
    for b, e in [(5, 5), (3, 11), (-1, 4)]:
        with pytest.raises(ValueError):
            check(lib.ipt_full_upload_columns(ctx.handle, n, dptr(d), None, dptr(delta), None, b, e, C.byref(h)))
