"""Single-eigenpair parity: dense GEMV and CSR SpMV paths on the B200 against
the reference's outputs (golden fixtures) and known answers
(proj/tests/test_solver.cpp:24-117, :217-253)."""
import math

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from conftest import golden
from paper_2012_14702_b200 import synth

pytestmark = pytest.mark.gpu


def explicit_2x2(eps):
    return ipt.Partition(np.array([0.0, 1.0]), np.array([[0.0, eps], [eps, 0.0]]))


def explicit_3x3(eps):
    return ipt.Partition(np.array([0.0, 1.0, 3.0]), eps * np.array([[0, 1, 2], [1, 0, 3], [2, 3, 0]], dtype=float))


def test_single_map_closed_form():
    """test_solver.cpp:25-32."""
    p = explicit_2x2(0.1)
    out = ipt.apply_map_single(p, ipt.build_gaps(p), 0, np.array([1.0, 0.0]))
    assert out[0] == 1.0 and out[1] == pytest.approx(-0.1, rel=1e-15)


def test_zero_residual_collapses_to_basis_vector():
    """test_solver.cpp:33-42 (complex iterate on a zero operator)."""
    p = ipt.Partition(np.array([0.0, 1.0, 2.0]), np.zeros((3, 3)))
    rng = np.random.default_rng(3)
    z = rng.standard_normal(3) + 1j * rng.standard_normal(3)
    z[1] = 1.0
    assert np.array_equal(ipt.apply_map_single(p, ipt.build_gaps(p), 1, z), [0, 1, 0])


def test_3x3_single_map_matches_reference(small):
    p = explicit_3x3(0.05)
    out = ipt.apply_map_single(p, ipt.build_gaps(p), 0, np.array([1.0, 0.0, 0.0]))
    assert np.max(np.abs(out - small["x3_0.05_map_single"])) <= 1e-15


@pytest.mark.parametrize("eps", [0.05, 0.1, 0.3, 1.0, 3.0])
def test_solve_single_2x2_matches_reference(small, eps):
    p = explicit_2x2(eps)
    r = ipt.solve_single(p, ipt.build_gaps(p), 0, ipt.IterationConfig(record_trace=True))
    meta = small[f"x2_{eps}_single_meta"]
    assert int(r.status) == int(meta[1])
    if r.status == ipt.SolveStatus.Converged:
        assert abs(r.iterations - int(meta[0])) <= 1
        assert np.max(np.abs(r.z - small[f"x2_{eps}_single_z"])) <= 1e-15
        assert r.eigenvalue == pytest.approx(meta[5], rel=1e-14)
    if eps == 0.1:  # closed form (test_solver.cpp:65-75)
        xs = (1.0 - math.sqrt(1.04)) / 0.2
        assert r.z[0] == 1.0
        assert r.z[1] == pytest.approx(xs, rel=1e-12)
        assert r.eigenvalue == pytest.approx(0.1 * xs, rel=1e-12)
        assert r.residual <= 1e-13
    if eps == 1.0:
        assert r.status != ipt.SolveStatus.Converged  # :84-88


def test_diagonal_matrix_converges_in_one_step():
    """test_solver.cpp:76-83."""
    p = ipt.Partition(np.array([0.0, 1.0]), np.zeros((2, 2)))
    r = ipt.solve_single(p, ipt.build_gaps(p), 1)
    assert r.status == ipt.SolveStatus.Converged and r.iterations == 1
    assert np.array_equal(r.z, [0.0, 1.0]) and r.eigenvalue == 1.0


def test_warm_start_renormalises_anchor():
    """test_solver.cpp:89-96."""
    p = explicit_2x2(0.05)
    r = ipt.solve_single(p, ipt.build_gaps(p), 0, warm_start=np.array([2.0, 0.1]))
    assert r.status == ipt.SolveStatus.Converged and r.z[0] == 1.0
    with pytest.raises(ValueError):
        ipt.solve_single(p, ipt.build_gaps(p), 0, warm_start=np.array([0.0, 0.1]))


def test_certified_instance_decays_geometrically():
    """test_solver.cpp:97-116 (complex random 12x12 scaled to a small coupling)."""
    rng = np.random.default_rng(5)
    m = rng.standard_normal((12, 12)) + 1j * rng.standard_normal((12, 12))
    p = ipt.partition(m)
    p = ipt.Partition(p.d, p.delta * 0.01)
    r = ipt.solve_single(p, ipt.build_gaps(p), 0, ipt.IterationConfig(record_trace=True))
    assert r.status == ipt.SolveStatus.Converged
    tr = np.array(r.trace)
    ratios = tr[1:-1] / tr[:-2]
    assert np.exp(np.mean(np.log(ratios))) < 1.0


def test_continuation_alpha_zero_reproduces_plain():
    """test_solver.cpp:218-227."""
    p = explicit_2x2(0.1)
    g = ipt.build_gaps(p)
    plain = ipt.solve_single(p, g, 0)
    cont = ipt.solve_single_continuation(p, g, 0, ipt.IterationConfig(), 0.0)
    assert cont.status == ipt.SolveStatus.Converged
    assert cont.iterations == plain.iterations + 1
    assert np.array_equal(cont.z, plain.z) and cont.eigenvalue == plain.eigenvalue


def test_continuation_zero_residual_any_alpha():
    """test_solver.cpp:228-238."""
    p = ipt.Partition(np.array([0.0, 1.0, 5.0]), np.zeros((3, 3)))
    g = ipt.build_gaps(p)
    for alpha in (0.0, 0.5, 0.9):
        r = ipt.solve_single_continuation(p, g, 2, ipt.IterationConfig(max_iterations=2000), alpha)
        assert r.status == ipt.SolveStatus.Converged and np.array_equal(r.z, [0, 0, 1])


def test_continuation_recovers_pinned_point(small):
    """test_solver.cpp:239-253 with kPinnedContinuationEps = -0.475 (fixtures.hpp:13)."""
    p = explicit_3x3(-0.475)
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(max_iterations=4000)
    assert ipt.solve_single(p, g, 1, cfg).status != ipt.SolveStatus.Converged
    c = ipt.solve_single_continuation(p, g, 1, cfg, 0.9)
    assert c.status == ipt.SolveStatus.Converged and c.residual <= 1e-8
    meta = small["x3_pinned_cont_meta"]
    assert abs(c.iterations - int(meta[0])) <= 1
    assert np.max(np.abs(c.z - small["x3_pinned_cont_z"])) <= 1e-12
    with pytest.raises(ValueError):
        ipt.solve_single_continuation(p, g, 1, cfg, 1.0)


def test_near_diagonal_singles_match_reference(small):
    for n, seed in ((8, 2024), (10, 7), (16, 8), (256, 9000)):
        key = f"nd_{n}_{seed}"
        p = ipt.partition(small[key + "_M"].real.copy())
        g = ipt.build_gaps(p)
        for j in (0, n // 2, n - 1):
            r = ipt.solve_single(p, g, j)
            meta = small[key + f"_single{j}_meta"]
            assert abs(r.iterations - int(meta[0])) <= 1
            assert np.max(np.abs(r.z - small[key + f"_single{j}_z"])) <= 1e-13
            assert r.eigenvalue == pytest.approx(meta[2], rel=1e-12)


def test_csr_matches_dense_path():
    p = synth.csr_ci(3000, 8, 0.01, 11)
    g = ipt.build_gaps(p, 0.0)
    dense = ipt.Partition(p.d, p.delta.to_dense())
    a = ipt.solve_single(p, g, 5, ipt.IterationConfig(tolerance=1e-12))
    b = ipt.solve_single(dense, g, 5, ipt.IterationConfig(tolerance=1e-12))
    assert a.iterations == b.iterations
    assert np.max(np.abs(a.z - b.z)) <= 1e-14
    assert a.eigenvalue == pytest.approx(b.eigenvalue, rel=1e-14)


def test_matvec_dense_and_csr_match_reference(port_arm):
    p = synth.csr_ci(5000, 16, 0.01, 12)
    rng = np.random.default_rng(4)
    x = rng.standard_normal(5000)
    y = ipt.kernels.matvec(p.delta, x)
    assert np.max(np.abs(y - port_arm.matvec(p.delta, x).real)) <= 1e-15
    a = rng.standard_normal((700, 700))
    assert np.max(np.abs(ipt.kernels.matvec(a, x[:700]) - a @ x[:700])) <= 1e-12
    xc = x[:700] + 1j * rng.standard_normal(700)
    assert np.max(np.abs(ipt.kernels.matvec(a, xc) - a @ xc)) <= 1e-12


# ----------------------------------------------------------------- configs 4 and 5


def test_config4_reduced_matches_reference():
    g = golden("single_configs.npz")
    p = synth.dense_normal(4096)
    r = ipt.solve_single(p, ipt.build_gaps(p), 0, ipt.IterationConfig(tolerance=1e-12))
    meta = g["c4_4096_meta"]
    assert r.status == ipt.SolveStatus.Converged and abs(r.iterations - int(meta[0])) <= 1
    assert r.eigenvalue == pytest.approx(meta[2], rel=1e-10)
    assert np.max(np.abs(r.z - g["c4_4096_z"])) <= 1e-9
    assert r.residual <= 1e-12


def test_config5_reduced_matches_reference():
    g = golden("single_configs.npz")
    n = 1 << 16
    p = synth.csr_ci(n)
    r = ipt.solve_single(p, ipt.build_gaps(p, 0.0), 0, ipt.IterationConfig(tolerance=1e-10))
    meta = g[f"c5_{n}_meta"]
    assert p.delta.nnz == int(meta[6])
    assert r.status == ipt.SolveStatus.Converged and abs(r.iterations - int(meta[0])) <= 1
    assert r.eigenvalue == pytest.approx(meta[2], rel=1e-10)
    assert np.max(np.abs(r.z - g[f"c5_{n}_z"])) <= 1e-9


@pytest.mark.slow
def test_config5_full_size():
    """N = 2^21 CI-like CSR: SURVEY §8(d) anchors (nnz, lambda_0) and the reference's iterate."""
    p = synth.config5()
    assert p.delta.nnz == 134216644
    with pytest.raises(ipt.DegenerateDiagonal):
        ipt.build_gaps(p)  # the default tolerance throws, as the reference does
    r = ipt.solve_single(p, ipt.build_gaps(p, 0.0), 0, ipt.IterationConfig(tolerance=1e-10))
    assert r.status == ipt.SolveStatus.Converged
    assert r.eigenvalue == pytest.approx(0.114060512572133, abs=1e-13)
    assert r.residual <= 1e-12
    g = golden("single_configs.npz")
    key = f"c5_{1 << 21}"
    if key + "_meta" in g.files:
        assert abs(r.iterations - int(g[key + "_meta"][0])) <= 1
        assert np.max(np.abs(r.z[g[key + "_zidx"]] - g[key + "_zval"])) <= 1e-9


@pytest.mark.slow
def test_config4_stand_in_n32768():
    """lambda_0 = 1.305492971741264 at the N = 32768 stand-in."""
    p = synth.dense_normal(32768)
    r = ipt.solve_single(p, ipt.build_gaps(p), 0, ipt.IterationConfig(tolerance=1e-12))
    assert r.status == ipt.SolveStatus.Converged
    assert r.eigenvalue == pytest.approx(1.305492971741264, abs=1e-13)
    g = golden("single_configs.npz")
    if "c4_32768_z" in g.files:
        assert np.max(np.abs(r.z - g["c4_32768_z"])) <= 1e-9
        assert abs(r.iterations - int(g["c4_32768_meta"][0])) <= 1


@pytest.mark.slow
def test_config4_full_size_n65536(port_arm):
    """BASELINE configs[3] at full size (34 GB operator): device vs the in-place CPU
    restatement of run_single (pinned bitwise to the reference at N = 4096)."""
    p = synth.config4()
    r = ipt.solve_single(p, ipt.build_gaps(p), 0, ipt.IterationConfig(tolerance=1e-12))
    o = port_arm.solve_single_real_dense(p.d, p.delta, 0, tol=1e-12)
    assert r.status == ipt.SolveStatus.Converged and o["status"] == 0
    assert abs(r.iterations - o["iterations"]) <= 1
    assert r.eigenvalue == pytest.approx(o["eigenvalue"], rel=1e-10)
    assert np.max(np.abs(r.z - o["z"])) <= 1e-9
    assert r.residual <= 1e-12 and r.z[0] == 1.0


# ----------------------------------------------------------------- Anderson mixing on the device


@pytest.mark.parametrize("name", ["acc7", "fci2k"])
@pytest.mark.parametrize("memory", [0, 2, 5])
def test_accelerated_matches_reference(name, memory):
    """solve_single_accelerated (anderson.cpp:184-247) on the acceptance #7 instance
    (gen_fci_like N=4096) and a second CI-like case, memory 0/2/5, against the reference."""
    g = golden("accelerated.npz")
    n = g[name + "_d"].size
    p = ipt.Partition(g[name + "_d"], ipt.CsrMatrix(n, n, g[name + "_rowptr"], g[name + "_cols"], g[name + "_vals"]))
    cfg = ipt.IterationConfig(residual_tolerance=1e-8, record_trace=True)
    r = ipt.solve_single_accelerated(p, ipt.build_gaps(p), 0, cfg, memory)
    meta = g[f"{name}_m{memory}_meta"]
    assert int(r.status) == int(meta[1]) == 0
    assert abs(r.matvec_count - int(meta[5])) <= 1
    assert r.residual <= 1e-8 / np.linalg.norm(r.z) * 1.0001
    assert r.eigenvalue == pytest.approx(meta[2], rel=1e-10)
    assert np.max(np.abs(r.z - g[f"{name}_m{memory}_z"])) <= 1e-9
    # memory 0 is the plain iteration with the residual stop (test_anderson.cpp:8-19)
    if memory == 0:
        plain = ipt.solve_single(p, ipt.build_gaps(p), 0, ipt.IterationConfig(tolerance=1e-12))
        assert r.eigenvalue == pytest.approx(plain.eigenvalue, rel=1e-9)
