"""Full-spectrum parity: the B200 path (C ABI -> DMMA kernels) against the
reference's outputs (golden fixtures made from the unmodified reference build)
and the CPU oracle, on the reference's own test cases (proj/tests/test_solver.cpp).

Tolerances (BASELINE.json north_star): eigenvalues 1e-10 relative, eigenvectors
1e-9 (both carry Z_jj = 1 exactly, so no sign normalisation is needed),
iterations within +-1 under the same stop rule, |MZ - Z Lambda|_F <= 1e-10 |M|_F.
"""
import math

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from conftest import golden
from paper_2012_14702_b200 import synth

pytestmark = pytest.mark.gpu

EPS = np.finfo(float).eps
LAM_REL = 1e-10
VEC_ABS = 1e-9


def explicit_2x2(eps):
    return ipt.Partition(np.array([0.0, 1.0]), np.array([[0.0, eps], [eps, 0.0]]))


def explicit_3x3(eps):
    return ipt.Partition(np.array([0.0, 1.0, 3.0]), eps * np.array([[0, 1, 2], [1, 0, 3], [2, 3, 0]], dtype=float))


def split(m):
    p = ipt.partition(np.asarray(m))
    if not np.any(np.asarray(p.delta).imag) and not np.any(np.asarray(p.d).imag):
        p = ipt.Partition(p.d.real.copy(), np.asarray(p.delta).real.copy())
    return p


def frob(p):
    return math.sqrt(np.sum(np.abs(ipt.reconstruct(p)) ** 2))


def test_context_is_b200():
    ctx = ipt.default_context()
    assert ctx.handle


# ----------------------------------------------------------------- maps


def test_identity_is_fixed_for_zero_residual():
    """test_solver.cpp:120-125."""
    p = ipt.Partition(np.array([0.0, 1.0, 2.0]), np.zeros((3, 3)))
    out = ipt.apply_map_full(p, ipt.build_gaps(p), np.eye(3))
    assert np.array_equal(out, np.eye(3))


def test_first_iterate_of_2x2(small):
    """test_solver.cpp:126-133: F(I) = [[1, 0.1], [-0.1, 1]]."""
    p = explicit_2x2(0.1)
    out = ipt.apply_map_full(p, ipt.build_gaps(p), np.eye(2))
    assert out[0, 0] == 1.0 and out[1, 1] == 1.0
    assert out[0, 1] == pytest.approx(0.1, rel=1e-15)
    assert out[1, 0] == pytest.approx(-0.1, rel=1e-15)
    assert np.max(np.abs(out - small["x2_0.1_map1"])) <= 1e-16


def test_complex_map_columns_equal_single_map(small):
    """test_solver.cpp:134-148 on the reference's complex random 6x6 inputs."""
    p = ipt.partition(small["cx6_M"])
    g = ipt.build_gaps(p)
    z = small["cx6_Zin"]
    full = ipt.apply_map_full(p, g, z)
    assert np.max(np.abs(full - small["cx6_F"])) <= 1e-13
    for j in range(6):
        ref = ipt.apply_map_single(p, g, j, z[:, j])
        assert np.max(np.abs(full[:, j] - ref)) <= 1e-12
    assert np.all(np.diag(full) == 1.0)  # unit diagonal is structural (:149-154)


# ----------------------------------------------------------------- solve_full: small


@pytest.mark.parametrize("eps", [0.05, 0.1, 0.3, 1.0, 3.0])
def test_solve_full_2x2_matches_reference(small, eps):
    p = explicit_2x2(eps)
    r = ipt.solve_full(p, ipt.build_gaps(p))
    meta = small[f"x2_{eps}_full_meta"]
    assert r.iterations == int(meta[0])
    assert int(r.status) == int(meta[1])
    if r.status != ipt.SolveStatus.Diverged:
        assert np.max(np.abs(r.Z - small[f"x2_{eps}_full_Z"])) <= 1e-15
        assert np.max(np.abs(r.eigenvalues - small[f"x2_{eps}_full_lam"])) <= 1e-15
        assert r.min_singular_value_estimate == pytest.approx(meta[3], rel=1e-9)
    if eps == 3.0:
        assert r.status == ipt.SolveStatus.Diverged  # test_solver.cpp:210-214


def test_zero_residual_one_iteration():
    """test_solver.cpp:174-180."""
    p = ipt.Partition(np.array([0.0, 1.0, 2.0]), np.zeros((3, 3)))
    r = ipt.solve_full(p, ipt.build_gaps(p))
    assert r.status == ipt.SolveStatus.Converged and r.iterations == 1
    assert np.array_equal(r.eigenvalues, [0.0, 1.0, 2.0])
    assert r.matmul_count == 2


@pytest.mark.parametrize("case", [(8, 2024), (10, 7), (16, 8), (256, 9000)])
@pytest.mark.parametrize("product", ["dmma", "ozaki"])
def test_solve_full_near_diagonal_matches_reference(small, case, product):
    """test_solver.cpp:158-209 instances (gen_near_diagonal, normal R), either FP64 product."""
    n, seed = case
    key = f"nd_{n}_{seed}"
    p = split(small[key + "_M"])
    cfg = ipt.IterationConfig(record_trace=True)
    r = ipt.solve_full(p, ipt.build_gaps(p), cfg, product=product)
    meta = small[key + "_meta"]
    assert abs(r.iterations - int(meta[0])) <= 1 and r.status == ipt.SolveStatus.Converged
    lam = small[key + "_lam"]
    assert np.max(np.abs(r.eigenvalues - lam) / np.abs(lam)) <= LAM_REL
    assert np.max(np.abs(r.Z - small[key + "_Z"])) <= VEC_ABS
    assert np.all(np.diag(r.Z) == 1.0)
    assert r.residual_frobenius <= 1e-10 * frob(p)
    assert r.min_singular_value_estimate == pytest.approx(meta[3], rel=1e-6)
    if key + "_direct" in small.files:  # direct-solver agreement (:167)
        direct = sorted(small[key + "_direct"], key=lambda z: z.real)
        got = sorted(r.eigenvalues, key=lambda z: z.real)
        assert max(abs(a - b) for a, b in zip(got, direct)) <= 1e-10
    trace = np.array(r.trace)
    ref_trace = small[key + "_trace"]
    k = min(len(trace), len(ref_trace))
    assert np.allclose(trace[: k - 1], ref_trace[: k - 1], rtol=1e-6, atol=1e-15)


def test_columns_of_solve_full_equal_solve_single(small):
    """test_solver.cpp:188-201 on the device, both sides through the C ABI."""
    p = split(small["nd_10_7_M"])
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig()
    full = ipt.solve_full(p, g, cfg)
    assert full.status == ipt.SolveStatus.Converged
    for j in (0, 4, 9):
        one = ipt.solve_single(p, g, j, cfg)
        assert one.status == ipt.SolveStatus.Converged
        assert np.max(np.abs(full.Z[:, j] - one.z)) <= 10 * cfg.tolerance


def test_converges_at_eps_03_uncertified():
    p = explicit_2x2(0.3)
    assert ipt.solve_full(p, ipt.build_gaps(p)).status == ipt.SolveStatus.Converged


def test_3x3_against_cubic_roots(small):
    """test_testgen.cpp:138-147."""
    p = explicit_3x3(0.05)
    r = ipt.solve_full(p, ipt.build_gaps(p))
    got = sorted(r.eigenvalues, key=lambda z: z.real)
    want = sorted(np.roots(np.poly(ipt.reconstruct(p))), key=lambda z: z.real)
    assert max(abs(a - b) for a, b in zip(got, want)) <= 1e-12
    assert np.max(np.abs(r.eigenvalues - small["x3_0.05_full_lam"])) <= 1e-14


def test_warm_start_renormalises_columns(small):
    p = split(small["nd_16_8_M"])
    g = ipt.build_gaps(p)
    ref = ipt.solve_full(p, g)
    warm = ref.Z * np.linspace(1.5, 2.5, 16)[None, :]
    r = ipt.solve_full(p, g, warm_start=warm)
    assert r.status == ipt.SolveStatus.Converged and r.iterations <= 2
    assert np.all(np.diag(r.Z) == 1.0)
    assert np.max(np.abs(r.Z - ref.Z)) <= 1e-13
    bad = warm.copy()
    bad[3, 3] = 0.0
    with pytest.raises(ValueError):
        ipt.solve_full(p, g, warm_start=bad)


def test_invalid_config_raises():
    p = explicit_2x2(0.1)
    g = ipt.build_gaps(p)
    for cfg in (ipt.IterationConfig(tolerance=0.0), ipt.IterationConfig(max_iterations=0),
                ipt.IterationConfig(divergence_threshold=1.0)):
        with pytest.raises(ValueError):
            ipt.solve_full(p, g, cfg)


def test_complex_certified_instances_converge_geometrically():
    """acceptance.cpp:74-108 style: complex d and complex Delta, scaled to a small coupling."""
    rng = np.random.default_rng(5)
    for n in (4, 9, 33, 64):
        delta = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * (0.02 / math.sqrt(n))
        np.fill_diagonal(delta, 0)
        d = np.arange(n) + 0.4j * rng.uniform(size=n)
        p = ipt.Partition(d, delta)
        cfg = ipt.IterationConfig(record_trace=True)
        r = ipt.solve_full(p, ipt.build_gaps(p), cfg)
        assert r.status == ipt.SolveStatus.Converged
        tr = np.array(r.trace)
        assert np.all(tr[1:] < tr[:-1]) or tr[-1] <= cfg.tolerance
        m = ipt.reconstruct(p)
        res = np.linalg.norm(m @ r.Z - r.Z * r.eigenvalues[None, :])
        assert res <= 1e-12 * np.linalg.norm(m)
        assert r.residual_frobenius == pytest.approx(res, rel=0.5, abs=1e-13)


@pytest.mark.parametrize("product", ["dmma", "ozaki"])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 33, 129, 200])
def test_odd_sizes_match_oracle(port_arm, n, product):
    """Arbitrary N (predicated tails, no CPU fallback) against the restatement, with
    either FP64 product."""
    rng = np.random.default_rng(n)
    delta = 0.05 * rng.uniform(-1, 1, (n, n))
    delta = 0.5 * (delta + delta.T)
    np.fill_diagonal(delta, 0)
    d = np.arange(1.0, n + 1)
    p = ipt.Partition(d, delta)
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-13), product=product)
    o = port_arm.solve_full(d, delta, tol=1e-13)
    assert abs(r.iterations - o["iterations"]) <= 1
    assert np.max(np.abs(r.eigenvalues - o["eigenvalues"].real) / np.abs(o["eigenvalues"].real)) <= LAM_REL
    assert np.max(np.abs(r.Z - o["Z"].real)) <= VEC_ABS
    assert r.min_singular_value_estimate == pytest.approx(o["sigma_min"], rel=1e-6)


def test_run_to_run_bitwise_deterministic():
    p = synth.dense_uniform(300, 0.01, 3)
    g = ipt.build_gaps(p)
    a = ipt.solve_full(p, g, ipt.IterationConfig(tolerance=1e-12))
    b = ipt.solve_full(p, g, ipt.IterationConfig(tolerance=1e-12))
    assert np.array_equal(a.Z, b.Z) and np.array_equal(a.eigenvalues, b.eigenvalues)
    assert a.residual_frobenius == b.residual_frobenius


# ----------------------------------------------------------------- config 1 (N = 1024)


@pytest.mark.parametrize("tag", ["rel_fro_tol12", "max_abs_tol12", "rel_fro_default"])
def test_config1_matches_reference(tag):
    g = golden("config1.npz")
    p = synth.config1()
    rule = "max_abs" if tag.startswith("max_abs") else "rel_fro"
    tol = 100 * EPS if tag.endswith("default") else 1e-12
    cfg = ipt.IterationConfig(tolerance=tol, stop_rule=rule, record_trace=True)
    r = ipt.solve_full(p, ipt.build_gaps(p), cfg)
    meta = g[tag + "_meta"]
    assert r.status == ipt.SolveStatus.Converged
    assert abs(r.iterations - int(meta[0])) <= 1
    lam = g[tag + "_lam"]
    assert np.max(np.abs(r.eigenvalues - lam) / np.abs(lam)) <= LAM_REL
    assert np.max(np.abs(r.Z[:, g["cols"]] - g[tag + "_cols"])) <= VEC_ABS
    assert r.residual_frobenius <= 1e-10 * frob(p)
    if tag == "rel_fro_tol12":
        assert r.min_singular_value_estimate == pytest.approx(meta[3], rel=1e-6)
    # SURVEY §8(d) anchors
    assert r.eigenvalues[0] == pytest.approx(0.999755195122348, abs=1e-13)
    assert r.eigenvalues[-1] == pytest.approx(1024.000266003840579, abs=1e-10)


# ----------------------------------------------------------------- kernels::matmul


def test_matmul_matches_reference_and_is_deterministic(small):
    """test_kernels.cpp:40-50 (<= 1e-13 |A||B|) and :69-83 (bitwise repeatable)."""
    for n in (1, 2, 3, 7, 16, 33, 64):
        a, b = small[f"mm_{n}_A"], small[f"mm_{n}_B"]
        c = ipt.kernels.matmul(a, b)
        scale = np.linalg.norm(a) * np.linalg.norm(b)
        assert np.max(np.abs(c - small[f"mm_{n}_C"])) <= 1e-13 * scale
        assert np.array_equal(c, ipt.kernels.matmul(a, b))
    rng = np.random.default_rng(3)
    a = rng.standard_normal((300, 170))
    b = rng.standard_normal((170, 260))
    assert np.max(np.abs(ipt.kernels.matmul(a, b) - a @ b)) <= 1e-13 * np.linalg.norm(a) * np.linalg.norm(b)


def test_matvec_identity_exact():
    """test_kernels.cpp:85-93."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal(17) + 1j * rng.standard_normal(17)
    assert np.array_equal(ipt.kernels.matvec(np.eye(17), x), x)


def test_sigma_min_matches_reference(ref_or_port_sigma=None):
    rng = np.random.default_rng(2)
    z = np.eye(40) + 0.05 * rng.standard_normal((40, 40))
    import oracle

    want = oracle.port().sigma_min(z)
    assert ipt.smallest_singular_value_estimate(z) == pytest.approx(want, rel=1e-8)
    zc = z + 0.03j * rng.standard_normal((40, 40))
    assert ipt.smallest_singular_value_estimate(zc) == pytest.approx(oracle.port().sigma_min(zc), rel=1e-8)
    assert ipt.smallest_singular_value_estimate(np.zeros((5, 5))) == 0.0


@pytest.mark.parametrize("n", [511, 640, 1100])
def test_sigma_min_across_cholesky_panels(port_arm, n):
    """sigma_min through the two-level blocked Cholesky (128-column sub-blocks inside
    512-column panels), sizes straddling the panel boundaries, against the oracle's
    partial-pivot LU route (solver.cpp:275-297)."""
    rng = np.random.default_rng(n)
    z = np.eye(n) + (0.3 / math.sqrt(n)) * rng.standard_normal((n, n))
    np.fill_diagonal(z, 1.0)
    want = port_arm.sigma_min(z)
    assert ipt.smallest_singular_value_estimate(z) == pytest.approx(want, rel=1e-8)


@pytest.mark.parametrize("n", [1, 130, 1000, 2100])
def test_identity_start_shortcut_is_bitwise_the_gemm_path(n):
    """F(I) is evaluated without the product (W = Delta I = Delta exactly) through K1's
    own epilogue; the whole solve must be bit-identical to running map 1 as a GEMM."""
    import os

    p = synth.config3(n=n) if n > 1 else ipt.Partition(np.array([1.0]), np.zeros((1, 1)))
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=1e-12, record_trace=True)
    a = ipt.solve_full(p, g, cfg)
    os.environ["IPT_IDENTITY_SHORTCUT"] = "0"
    try:
        b = ipt.solve_full(p, g, cfg)
    finally:
        del os.environ["IPT_IDENTITY_SHORTCUT"]
    assert a.iterations == b.iterations and a.trace == b.trace
    assert np.array_equal(a.Z, b.Z) and np.array_equal(a.eigenvalues, b.eigenvalues)
    assert a.residual_frobenius == b.residual_frobenius
    assert a.min_singular_value_estimate == b.min_singular_value_estimate


def test_identity_start_with_nonfinite_delta_matches_gemm_semantics():
    """An Inf in Delta makes the GEMM's zero terms NaN; the shortcut is disabled then."""
    n = 64
    d = np.arange(n, dtype=float)
    delta = np.zeros((n, n))
    delta[3, 7] = np.inf
    r = ipt.solve_full(ipt.Partition(d, delta), ipt.build_gaps(ipt.Partition(d, delta)))
    assert r.status == ipt.SolveStatus.Diverged and r.iterations == 1


def test_divergence_status_and_step_match_oracle(port_arm):
    """A strongly perturbed instance: divergence is tested before convergence
    (solver.cpp:241-249) and reported at the same iteration as the restatement."""
    n = 96
    rng = np.random.default_rng(4)
    delta = 2.0 * rng.uniform(-1, 1, (n, n))
    delta = 0.5 * (delta + delta.T)
    np.fill_diagonal(delta, 0)
    d = np.arange(1.0, n + 1)
    p = ipt.Partition(d, delta)
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(divergence_threshold=1e6), want_sigma_min=False)
    o = port_arm.solve_full(d, delta, div_thr=1e6, sigma=False)
    assert int(r.status) == o["status"] == int(ipt.SolveStatus.Diverged)
    assert r.iterations == o["iterations"]


@pytest.mark.parametrize("max_iter", [1, 2, 3])
def test_max_iterations_returns_the_last_iterate(port_arm, max_iter):
    n = 150
    p = synth.dense_uniform(n, 0.3 / np.sqrt(n), 5)
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(max_iterations=max_iter, tolerance=1e-15))
    o = port_arm.solve_full(p.d, p.delta, tol=1e-15, max_iter=max_iter)
    assert r.status == ipt.SolveStatus.MaxIterations and int(o["status"]) == 1
    assert r.iterations == o["iterations"] == max_iter
    assert r.matmul_count == o["matmul_count"] == max_iter + 1
    assert np.max(np.abs(r.Z - o["Z"].real)) <= VEC_ABS
    np.testing.assert_allclose(r.eigenvalues, o["eigenvalues"].real, rtol=LAM_REL, atol=0)


def test_empty_problem_is_rejected():
    p = ipt.Partition(np.zeros(0), np.zeros((0, 0)))
    with pytest.raises(ValueError):
        ipt.solve_full(p, ipt.build_gaps(p))
