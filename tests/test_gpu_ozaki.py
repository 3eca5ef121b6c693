"""FP64-accurate products on the tcgen05 INT8 datapath (Ozaki scheme II, ozaki.cu): the
INT8 GEMM is exact, and the full-spectrum solve with product='ozaki' matches the DMMA
solve (and therefore the reference) far inside the north_star tolerances."""
import ctypes as C
import math
import os

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from conftest import golden
from paper_2012_14702_b200 import _lib, synth
from paper_2012_14702_b200._lib import check

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(128, 256, 128), (256, 512, 1024), (384, 768, 2176)])
def test_i8_gemm_is_exact(shape):
    M, N, K = shape
    rng = np.random.default_rng(M + N + K)
    a = rng.integers(-128, 128, (M, K), dtype=np.int8)
    b = rng.integers(-128, 128, (N, K), dtype=np.int8)
    c = np.empty((M, N), np.int32)
    ms = C.c_double()
    ctx = ipt.default_context()
    check(_lib.load().ipt_i8_gemm(ctx.handle, M, N, K, a.ctypes.data, b.ctypes.data, c.ctypes.data, 0, C.byref(ms)))
    assert np.array_equal(c, a.astype(np.int64) @ b.astype(np.int64).T)


@pytest.mark.parametrize("kind", ["1sm", "mc", "2sm", "2sm512"])
@pytest.mark.parametrize("group", ["1", "3", "8", "1000"])
def test_i8_gemm_kernel_variants_are_exact(kind, group, monkeypatch):
    """Every tile schedule (one SM, B multicast over a CTA pair, cta_group::2 with
    256 x 256 and 256 x 512 pair tiles) under every rasterisation grouping (including a
    ragged last group) gives the exact int32 product."""
    monkeypatch.setenv("IPT_I8_KERNEL", kind)
    monkeypatch.setenv("IPT_I8_GROUP", group)
    M, N, K = 1280, 1024, 640
    rng = np.random.default_rng(7)
    a = rng.integers(-128, 128, (M, K), dtype=np.int8)
    b = rng.integers(-128, 128, (N, K), dtype=np.int8)
    c = np.empty((M, N), np.int32)
    ctx = ipt.default_context()
    check(_lib.load().ipt_i8_gemm(ctx.handle, M, N, K, a.ctypes.data, b.ctypes.data, c.ctypes.data, 0, None))
    assert np.array_equal(c, a.astype(np.int64) @ b.astype(np.int64).T)


def _row_exponents(x):
    """52 - ilogb(row max): the row scaling of ozaki.cu's exponent_kernel (None: non-finite)."""
    out = []
    for row in x:
        mx = float(np.max(np.abs(row))) if row.size else 0.0
        out.append(None if not math.isfinite(mx) else 0 if mx == 0.0 else 52 - (math.frexp(mx)[1] - 1))
    return out


def _exact_ozaki(a, bt):
    """C_ij = the correctly rounded exact dot product of row i of A and row j of B^T, both
    scaled to 53-bit integers, scaled back: Python integers, CPython's correctly rounded
    int -> float, and ldexp (exact but for subnormal results)."""
    ea, eb = _row_exponents(a), _row_exponents(bt)

    def ints(x, e):
        return np.array([[int(np.rint(math.ldexp(float(v), e[i]))) if e[i] is not None else 0 for v in x[i]]
                         for i in range(x.shape[0])], dtype=object).reshape(x.shape)

    p = ints(a, ea).dot(ints(bt, eb).T) if a.shape[1] else np.zeros((a.shape[0], bt.shape[0]), dtype=object)
    c = np.empty(p.shape)
    for i in range(p.shape[0]):
        for j in range(p.shape[1]):
            c[i, j] = math.nan if ea[i] is None or eb[j] is None else math.ldexp(float(p[i, j]), -(ea[i] + eb[j]))
    return c


@pytest.mark.parametrize("m,n,k", [(70, 45, 300), (33, 130, 2000), (1, 1, 1), (5, 7, 0)])
def test_ozaki_dgemm_is_the_rounded_exact_product(m, n, k):
    """Bitwise: the Garner reconstruction, the 128-bit Horner sum and the int128 -> FP64
    rounding reproduce the exact integer product of the scaled operands, rounded once."""
    rng = np.random.default_rng(m * 1000 + n + k)
    a = rng.standard_normal((m, k)) * np.exp2(rng.integers(-40, 40, (m, 1)))
    b = rng.standard_normal((k, n)) * np.exp2(rng.integers(-40, 40, (1, n)))
    if k > 4:
        a[0, :3] *= 2.0 ** -45  # far below the row max: truncated by the 53-bit scaling
        b[1, -1] = 0.0
    if m > 3:
        a[2] = 0.0  # zero row
    c = ipt.kernels.matmul_ozaki(a, b)
    ref = _exact_ozaki(a, np.ascontiguousarray(b.T))
    assert c.shape == (m, n)
    assert np.array_equal(c.view(np.int64), ref.view(np.int64)), np.max(np.abs(c - ref))
    if k:
        bound = 4 * k * np.finfo(float).eps * (np.abs(a) @ np.abs(b))
        assert np.all(np.abs(c - a @ b) <= bound + 1e-300)


def test_ozaki_dgemm_nonfinite_rows_give_nan():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((9, 50))
    b = rng.standard_normal((50, 6))
    a[4, 7] = np.inf
    b[3, 2] = np.nan
    c = ipt.kernels.matmul_ozaki(a, b)
    assert np.all(np.isnan(c[4, :])) and np.all(np.isnan(c[:, 2]))
    mask = np.ones_like(c, bool)
    mask[4, :] = False
    mask[:, 2] = False
    assert np.all(np.isfinite(c[mask]))
    with np.errstate(invalid="ignore"):
        ref = a @ b
    assert np.allclose(c[mask], ref[mask], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("n", [64, 300, 1000, 2048])
def test_ozaki_solve_matches_dmma(n):
    p = synth.dense_uniform(n, 0.3 / np.sqrt(n), 11)
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=1e-13)
    a = ipt.solve_full(p, g, cfg, product="dmma")
    b = ipt.solve_full(p, g, cfg, product="ozaki")
    assert a.iterations == b.iterations and a.status == b.status
    assert np.max(np.abs(a.eigenvalues - b.eigenvalues) / np.abs(a.eigenvalues)) <= 1e-14
    assert np.max(np.abs(a.Z - b.Z)) <= 1e-13
    assert b.residual_frobenius <= 10 * max(a.residual_frobenius, 1e-14)


def test_ozaki_one_map_from_a_dense_warm_start():
    """A map of a general Z (not the converged basis): entries over many binades."""
    n = 700
    rng = np.random.default_rng(5)
    p = synth.dense_uniform(n, 0.3 / np.sqrt(n), 12)
    g = ipt.build_gaps(p)
    z = np.eye(n) + rng.standard_normal((n, n)) * np.exp(rng.uniform(-20, 2, (n, n)))
    np.fill_diagonal(z, 1.0)
    cfg = ipt.IterationConfig(max_iterations=1, divergence_threshold=1e300)
    a = ipt.solve_full(p, g, cfg, warm_start=z, want_sigma_min=False, product="dmma")
    b = ipt.solve_full(p, g, cfg, warm_start=z, want_sigma_min=False, product="ozaki")
    scale = np.max(np.abs(a.Z), axis=0)
    assert np.max(np.abs(a.Z - b.Z) / scale) <= 1e-14


def test_ozaki_is_bitwise_deterministic():
    p = synth.dense_uniform(512, 0.01, 3)
    g = ipt.build_gaps(p)
    a = ipt.solve_full(p, g, product="ozaki")
    b = ipt.solve_full(p, g, product="ozaki")
    assert np.array_equal(a.Z, b.Z) and np.array_equal(a.eigenvalues, b.eigenvalues)


def test_ozaki_nonfinite_delta_falls_back():
    n = 64
    d = np.arange(n, dtype=float)
    delta = np.zeros((n, n))
    delta[3, 7] = np.inf
    p = ipt.Partition(d, delta)
    r = ipt.solve_full(p, ipt.build_gaps(p), product="ozaki")
    assert r.status == ipt.SolveStatus.Diverged and r.iterations == 1


# ------------------------------------------------ parity with the reference (golden fixtures)


def _frob(p):
    return math.sqrt(np.sum(p.delta ** 2) + np.sum(p.d ** 2))


@pytest.mark.parametrize("tag", ["rel_fro_tol12", "max_abs_tol12", "rel_fro_default"])
def test_ozaki_config1_matches_reference(tag):
    """configs[0] (N = 1024) with W = Delta Z by Ozaki scheme II against the reference
    build's own solve_full (tests/golden/config1.npz), north_star tolerances."""
    g = golden("config1.npz")
    p = synth.config1()
    rule = "max_abs" if tag.startswith("max_abs") else "rel_fro"
    tol = 100 * np.finfo(float).eps if tag.endswith("default") else 1e-12
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=tol, stop_rule=rule), product="ozaki")
    meta = g[tag + "_meta"]
    assert r.status == ipt.SolveStatus.Converged
    assert abs(r.iterations - int(meta[0])) <= 1
    lam = g[tag + "_lam"]
    assert np.max(np.abs(r.eigenvalues - lam) / np.abs(lam)) <= 1e-10
    assert np.max(np.abs(r.Z[:, g["cols"]] - g[tag + "_cols"])) <= 1e-9
    assert r.residual_frobenius <= 1e-10 * _frob(p)
    assert np.all(np.diag(r.Z) == 1.0)


def test_ozaki_config2_matches_reference_columns():
    """configs[1] (N = 8192): columns of the reference's solve_single(j) (the column route
    of SURVEY 8c, tests/golden/full_columns.npz) and the SURVEY 8(d) anchor."""
    p = synth.config2()
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12), product="ozaki")
    assert r.status == ipt.SolveStatus.Converged and abs(r.iterations - 5) <= 1
    assert r.eigenvalues[0] == pytest.approx(0.999960499073907, abs=1e-13)
    assert r.residual_frobenius <= 1e-10 * _frob(p)
    g = golden("full_columns.npz")
    cols, lam = g["n8192_cols"], g["n8192_lam"]
    assert np.max(np.abs(r.eigenvalues[cols] - lam) / np.abs(lam)) <= 1e-10
    assert np.max(np.abs(r.Z[:, cols] - g["n8192_z"])) <= 1e-9


# ------------------------------------- diagonal split: fewer moduli, the same exact product


def _moduli_after_maps(p, maps, warm=None):
    lib = _lib.load()
    ctx = ipt.default_context()
    n = len(p.d)
    h = C.c_void_p()
    check(lib.ipt_full_upload(ctx.handle, n, _lib.dptr(p.d), None, _lib.dptr(np.ascontiguousarray(p.delta)), None,
                              C.byref(h)))
    try:
        check(lib.ipt_full_reset(ctx.handle, h, _lib.dptr(warm), None))
        check(lib.ipt_full_set_product(h, _lib.PRODUCT_OZAKI))
        tot, ker = C.c_double(), C.c_double()
        check(lib.ipt_full_run_maps(ctx.handle, h, maps, C.byref(tot), C.byref(ker)))
        m = C.c_int32()
        check(lib.ipt_full_ozaki_moduli(h, C.byref(m)))
        return m.value
    finally:
        lib.ipt_full_free(h)


def test_split_needs_fewer_moduli_on_the_ipt_iterates():
    """Z_jj = 1 split off: the IPT iterates' off-diagonal column norms need 13 moduli at the
    config-3 construction (|Y_j|_1 ~ 0.04); a dense O(1) warm start needs 15-16
    (|Y'_j|_1 ~ n 2^51 > 2^61)."""
    n = 2048
    p = synth.dense_uniform(n, 0.32 / np.sqrt(n), 21)
    assert _moduli_after_maps(p, 3) <= 13
    rng = np.random.default_rng(4)
    warm = np.eye(n) + rng.standard_normal((n, n))
    np.fill_diagonal(warm, 1.0)
    assert _moduli_after_maps(p, 1, np.ascontiguousarray(warm)) >= 15


@pytest.mark.parametrize("n", [300, 1000, 2049])
def test_split_is_bitwise_the_16_moduli_product(n, monkeypatch):
    """The split product (fewer moduli + the diagonal term added in 128-bit integers) is the
    same correctly rounded exact product: solves agree bit for bit with IPT_OZAKI_SPLIT=0."""
    p = synth.dense_uniform(n, 0.3 / np.sqrt(n), 31)
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=1e-13)
    a = ipt.solve_full(p, g, cfg, product="ozaki")
    monkeypatch.setenv("IPT_OZAKI_SPLIT", "0")
    b = ipt.solve_full(p, g, cfg, product="ozaki")
    assert a.iterations == b.iterations
    assert np.array_equal(a.Z, b.Z) and np.array_equal(a.eigenvalues, b.eigenvalues)
    assert a.residual_frobenius == b.residual_frobenius


def test_split_is_bitwise_on_a_nonsymmetric_delta_and_wide_warm_start(monkeypatch):
    """Delta_ij for the diagonal term comes from the transposed copy (nonsymmetric Delta),
    and a warm start whose columns span many binades (Z'_jj not a power of two)."""
    n = 700
    rng = np.random.default_rng(9)
    d = np.arange(1.0, n + 1.0)
    delta = 0.01 * rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(delta, 0.0)
    p = ipt.Partition(d, delta)
    g = ipt.build_gaps(p)
    z = np.eye(n) + rng.standard_normal((n, n)) * np.exp(rng.uniform(-20, 0, (n, n)))
    np.fill_diagonal(z, 1.0)
    cfg = ipt.IterationConfig(max_iterations=2, divergence_threshold=1e300)
    a = ipt.solve_full(p, g, cfg, warm_start=z, want_sigma_min=False, product="ozaki")
    monkeypatch.setenv("IPT_OZAKI_SPLIT", "0")
    b = ipt.solve_full(p, g, cfg, warm_start=z, want_sigma_min=False, product="ozaki")
    assert np.array_equal(a.Z, b.Z) and np.array_equal(a.eigenvalues, b.eigenvalues)


# ------------------------------------------------------------- complex inputs (3M)


@pytest.mark.parametrize("n", [4, 33, 64, 300, 700])
def test_ozaki_complex_matches_dmma(n):
    """Complex d and Delta (acceptance.cpp:80-88 style): the 3M product with each real
    product by Ozaki scheme II agrees with the DMMA 3M product and with the direct check."""
    rng = np.random.default_rng(n + 7)
    delta = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * (0.02 / math.sqrt(n))
    np.fill_diagonal(delta, 0)
    d = np.arange(n) + 0.4j * rng.uniform(size=n)
    p = ipt.Partition(d, delta)
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=1e-13)
    a = ipt.solve_full(p, g, cfg, product="dmma")
    b = ipt.solve_full(p, g, cfg, product="ozaki")
    assert b.status == ipt.SolveStatus.Converged and a.iterations == b.iterations
    assert np.max(np.abs(a.eigenvalues - b.eigenvalues) / np.abs(a.eigenvalues)) <= 1e-13
    assert np.max(np.abs(a.Z - b.Z)) <= 1e-13
    m = ipt.reconstruct(p)
    res = np.linalg.norm(m @ b.Z - b.Z * b.eigenvalues[None, :])  # (host rounding of d_i z dominates)
    assert res <= 1e-12 * np.linalg.norm(m)
    # the device residual is the reference's |d_i Z_ij + W_ij - Z_ij Lambda_j| form
    assert b.residual_frobenius <= 10 * max(a.residual_frobenius, 1e-15)


def test_ozaki_complex_uses_fewer_than_16_moduli():
    n = 1024
    rng = np.random.default_rng(3)
    delta = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * (0.02 / math.sqrt(n))
    np.fill_diagonal(delta, 0)
    d = np.arange(n) + 0.4j * rng.uniform(size=n)
    lib = _lib.load()
    ctx = ipt.default_context()
    h = C.c_void_p()
    dr, di = np.ascontiguousarray(delta.real), np.ascontiguousarray(delta.imag)
    check(lib.ipt_full_upload(ctx.handle, n, _lib.dptr(np.ascontiguousarray(d.real)),
                              _lib.dptr(np.ascontiguousarray(d.imag)), _lib.dptr(dr), _lib.dptr(di), C.byref(h)))
    try:
        check(lib.ipt_full_reset(ctx.handle, h, None, None))
        check(lib.ipt_full_set_product(h, _lib.PRODUCT_OZAKI))
        tot, ker = C.c_double(), C.c_double()
        check(lib.ipt_full_run_maps(ctx.handle, h, 3, C.byref(tot), C.byref(ker)))
        m = C.c_int32()
        check(lib.ipt_full_ozaki_moduli(h, C.byref(m)))
        assert 9 <= m.value <= 15
    finally:
        lib.ipt_full_free(h)
