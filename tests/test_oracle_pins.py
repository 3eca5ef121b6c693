"""Pin the CPU oracle before trusting it (CPU only, no GPU).

The restatement (oracle/ipt_oracle.c) is checked against
  * the reference's own outputs, committed as golden fixtures by
    tests/golden/make_golden.py from the unmodified reference build;
  * the reference's known answers (proj/tests/test_solver.cpp, test_testgen.cpp);
  * the sanity anchors recorded from the reference in SURVEY.md §8(d);
  * the reference build itself when oracle/_ref is present (this container).
"""
import math

import numpy as np
import pytest

from conftest import golden
from paper_2012_14702_b200 import synth

EPS = np.finfo(float).eps


def explicit_2x2(eps):  # proj/src/testgen.cpp:196-201
    return np.array([0.0, 1.0]), np.array([[0.0, eps], [eps, 0.0]], dtype=complex)


def explicit_3x3(eps):  # proj/src/testgen.cpp:203-210
    return np.array([0.0, 1.0, 3.0]), complex(eps) * np.array([[0, 1, 2], [1, 0, 3], [2, 3, 0]], dtype=complex)


def split(m):
    d = np.diag(m).copy()
    delta = m.copy()
    np.fill_diagonal(delta, 0)
    return d, delta


def bitwise(a, b):
    return np.array_equal(np.asarray(a, np.complex128).view(np.float64), np.asarray(b, np.complex128).view(np.float64))


# ---------------------------------------------------------------- generator


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_rng_matches_reference_stream(ref_arm, kind):
    for stream in (0, 1, 2, 7):
        a = ref_arm.rng_draws(42, kind, 2000, stream=stream)
        b = synth.rng_draws(42, kind, 2000, stream=stream)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_rng_below_matches_reference(ref_arm):
    a = ref_arm.rng_draws(42, 3, 5000, stream=1, bound=1 << 21)
    b = synth.rng_draws(42, 3, 5000, stream=1, bound=1 << 21)
    assert np.array_equal(a, b)


def test_rng_first_draws_are_pinned():
    """Pinned values of xoshiro256++/splitmix64 (rng.hpp) for seed 42, stream 0."""
    u = synth.rng_draws(42, 1, 3, stream=0)
    assert u.tolist() == pytest.approx([0.22821139, 0.7847751, 0.16243346], abs=5e-9)


# ---------------------------------------------------------------- kernels


def test_port_gemm_bitwise_equals_reference(small, port_arm):
    for n in (1, 2, 3, 7, 16, 33, 64):
        c = port_arm.gemm(small[f"mm_{n}_A"], small[f"mm_{n}_B"])
        assert bitwise(c, small[f"mm_{n}_C"]), n


def test_port_matvec_matches_reference(ref_arm, port_arm):
    rng = np.random.default_rng(1)
    a = rng.standard_normal((40, 40)) + 1j * rng.standard_normal((40, 40))
    x = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    assert np.max(np.abs(port_arm.matvec(a, x) - ref_arm.matvec(a, x))) <= 1e-13
    p = synth.csr_ci(4096, 8, 0.01, 3)
    xr = rng.standard_normal(4096)
    assert np.max(np.abs(port_arm.matvec(p.delta, xr) - ref_arm.matvec(p.delta, xr))) <= 1e-15


# ---------------------------------------------------------------- known answers


def test_known_answer_2x2_single_map(port_arm):
    """test_solver.cpp:25-32: f_0((1,0)) on the 2x2 family at eps=0.1 is (1, -0.1)."""
    d, delta = explicit_2x2(0.1)
    r = port_arm.solve_single(d, delta, 0, max_iter=1)
    assert r["z"][0] == 1.0
    assert r["z"][1].real == pytest.approx(-0.1, rel=1e-15)


def test_known_answer_2x2_fixed_point(port_arm):
    """test_solver.cpp:65-75: x* = (1 - sqrt(1.04))/0.2, lambda = 0.1 x*, residual <= 1e-13."""
    d, delta = explicit_2x2(0.1)
    r = port_arm.solve_single(d, delta, 0)
    xs = (1.0 - math.sqrt(1.04)) / 0.2
    assert r["status"] == 0
    assert r["z"][1].real == pytest.approx(xs, rel=1e-12)
    assert r["eigenvalue"].real == pytest.approx(0.1 * xs, rel=1e-12)
    assert r["residual"] <= 1e-13


def test_known_answer_full_first_iterate(port_arm):
    """test_solver.cpp:126-133: F(I) on the 2x2 family = [[1, 0.1], [-0.1, 1]]."""
    d, delta = explicit_2x2(0.1)
    f, _ = port_arm.full_map_block(d, delta, 0, np.eye(2))
    assert f[0, 0] == 1 and f[1, 1] == 1
    assert f[0, 1].real == pytest.approx(0.1, rel=1e-15)
    assert f[1, 0].real == pytest.approx(-0.1, rel=1e-15)


def test_known_answer_3x3_cubic_roots(port_arm):
    """test_testgen.cpp:138-147: eigenvalues against the characteristic polynomial (1e-12)."""
    d, delta = explicit_3x3(0.05)
    r = port_arm.solve_full(d, delta)
    m = np.diag(d).astype(complex) + delta
    roots = np.roots(np.poly(m))
    got = sorted(r["eigenvalues"], key=lambda z: z.real)
    want = sorted(roots, key=lambda z: z.real)
    assert max(abs(a - b) for a, b in zip(got, want)) <= 1e-12


def test_known_answer_divergence_and_zero_delta(port_arm):
    """test_solver.cpp:174-180, :210-214."""
    d, delta = explicit_2x2(3.0)
    assert port_arm.solve_full(d, delta)["status"] == 2
    r = port_arm.solve_full(np.array([0.0, 1.0, 2.0]), np.zeros((3, 3)))
    assert r["status"] == 0 and r["iterations"] == 1
    assert np.array_equal(r["eigenvalues"], [0, 1, 2])


def test_known_answer_continuation(port_arm):
    """test_solver.cpp:218-227 (alpha = 0: plain + 1 iterations) and :239-253 (pinned eps)."""
    d, delta = explicit_2x2(0.1)
    plain = port_arm.solve_single(d, delta, 0)
    cont = port_arm.solve_single(d, delta, 0, mode="continuation", alpha=0.0)
    assert cont["iterations"] == plain["iterations"] + 1
    assert bitwise(cont["z"], plain["z"])
    d, delta = explicit_3x3(-0.475)  # fixtures.hpp:13
    assert port_arm.solve_single(d, delta, 1, max_iter=4000)["status"] != 0
    c = port_arm.solve_single(d, delta, 1, max_iter=4000, mode="continuation", alpha=0.9)
    assert c["status"] == 0 and c["residual"] <= 1e-8


# ---------------------------------------------------------------- against the reference's outputs


@pytest.mark.parametrize("eps", [0.05, 0.1, 0.3, 1.0, 3.0])
def test_port_2x2_equals_reference(small, port_arm, eps):
    d, delta = explicit_2x2(eps)
    s = port_arm.solve_single(d, delta, 0)
    meta = small[f"x2_{eps}_single_meta"]
    assert s["iterations"] == int(meta[0]) and s["status"] == int(meta[1])
    assert bitwise(s["z"], small[f"x2_{eps}_single_z"])
    f = port_arm.solve_full(d, delta)
    fm = small[f"x2_{eps}_full_meta"]
    assert f["iterations"] == int(fm[0]) and f["status"] == int(fm[1])
    if f["status"] != 2:
        assert bitwise(f["Z"], small[f"x2_{eps}_full_Z"])
        assert bitwise(f["eigenvalues"], small[f"x2_{eps}_full_lam"])


@pytest.mark.parametrize("case", [(8, 2024), (10, 7), (16, 8), (256, 9000)])
def test_port_near_diagonal_equals_reference(small, port_arm, case):
    n, seed = case
    key = f"nd_{n}_{seed}"
    d, delta = split(small[key + "_M"])
    r = port_arm.solve_full(d, delta)
    meta = small[key + "_meta"]
    assert r["iterations"] == int(meta[0]) and r["status"] == int(meta[1])
    # complex arithmetic: the reference's g++ contracts into FMAs where the C port does not
    assert np.max(np.abs(r["Z"] - small[key + "_Z"])) <= 1e-14
    assert np.max(np.abs(r["eigenvalues"] - small[key + "_lam"]) / np.abs(small[key + "_lam"])) <= 1e-14
    assert r["residual_frobenius"] == pytest.approx(meta[2], rel=0.5, abs=1e-14)
    assert r["sigma_min"] == pytest.approx(meta[3], rel=1e-10)
    for j in (0, n // 2, n - 1):
        s = port_arm.solve_single(d, delta, j)
        assert np.max(np.abs(s["z"] - small[key + f"_single{j}_z"])) <= 1e-14


def test_port_complex_map_equals_reference(small, port_arm):
    d, delta = split(small["cx6_M"])
    f, _ = port_arm.full_map_block(d, delta, 0, small["cx6_Zin"])
    assert np.max(np.abs(f - small["cx6_F"])) <= 1e-14
    # columns of the full map equal the anchored single map (test_solver.cpp:134-148)
    assert np.max(np.abs(f - small["cx6_single"])) <= 1e-12


@pytest.mark.parametrize("tag", ["rel_fro_tol12", "max_abs_tol12", "rel_fro_default"])
def test_port_config1_bitwise_equals_reference(port_arm, tag):
    """Config 1 (N=1024): the restatement reproduces the reference bit for bit."""
    g = golden("config1.npz")
    p = synth.config1()
    rule = "max_abs" if tag.startswith("max_abs") else "rel_fro"
    tol = 100 * EPS if tag.endswith("default") else 1e-12
    r = port_arm.solve_full(p.d, p.delta, tol=tol, stop_rule=rule, sigma=(tag == "rel_fro_tol12"))
    meta = g[tag + "_meta"]
    assert r["iterations"] == int(meta[0]) and r["status"] == int(meta[1])
    assert np.array_equal(r["eigenvalues"].real, g[tag + "_lam"])
    assert np.array_equal(r["Z"].real[:, g["cols"]], g[tag + "_cols"])
    if rule == "rel_fro":  # the max-abs driver sums its residual in its own (serial) order
        assert r["residual_frobenius"] == meta[2]
    else:
        assert r["residual_frobenius"] == pytest.approx(meta[2], rel=1e-12)
    if tag == "rel_fro_tol12":
        assert r["sigma_min"] == meta[3]


def test_config1_survey_anchors():
    """Lambda_0 = 0.999755195122348, Lambda_{N-1} = 1024.000266003840579."""
    g = golden("config1.npz")
    lam = g["rel_fro_default_lam"]
    assert lam[0] == pytest.approx(0.999755195122348, abs=2e-15)
    assert lam[-1] == pytest.approx(1024.000266003840579, abs=1e-12)
    assert int(g["rel_fro_default_meta"][0]) == 8  # 8 iterations at the default tolerance


def test_single_configs_reduced_port_vs_reference(port_arm):
    g = golden("single_configs.npz")
    p = synth.dense_normal(4096)
    r = port_arm.solve_single(p.d, p.delta, 0, tol=1e-12)
    meta = g["c4_4096_meta"]
    assert r["iterations"] == int(meta[0])
    assert r["eigenvalue"].real == pytest.approx(meta[2], rel=1e-14)
    assert np.max(np.abs(r["z"].real - g["c4_4096_z"])) <= 1e-15
    p = synth.csr_ci(1 << 16)
    r = port_arm.solve_single(p.d, p.delta, 0, tol=1e-10)
    meta = g[f"c5_{1 << 16}_meta"]
    assert r["iterations"] == int(meta[0]) and p.delta.nnz == int(meta[6])
    assert r["eigenvalue"].real == pytest.approx(meta[2], rel=1e-14)
    assert np.max(np.abs(r["z"].real - g[f"c5_{1 << 16}_z"])) <= 1e-15


def test_survey_anchor_config5_full_size():
    """config 5 has nnz = 134,216,644 and lambda_0 = 0.114060512572133."""
    g = golden("single_configs.npz")
    key = f"c5_{1 << 21}_meta"
    if key not in g:
        pytest.skip("full-size config 5 golden not generated (make_golden.py --big)")
    meta = g[key]
    assert int(meta[6]) == 134216644
    assert meta[2] == pytest.approx(0.114060512572133, abs=1e-14)


def test_port_real_dense_single_bitwise_equals_reference(port_arm):
    """The in-place real restatement (used for config 4 at N = 65536) reproduces the
    reference's complex solve_single bit for bit on real inputs."""
    g = golden("single_configs.npz")
    p = synth.dense_normal(4096)
    r = port_arm.solve_single_real_dense(p.d, p.delta, 0, tol=1e-12)
    meta = g["c4_4096_meta"]
    assert r["iterations"] == int(meta[0]) and r["status"] == int(meta[1])
    assert np.array_equal(r["z"], g["c4_4096_z"])
    assert r["eigenvalue"] == meta[2]


def test_config3_iteration_pin_fixture_is_decisive():
    """tests/golden/config3_trace.npz (make_config3_trace.py: the reference loop restated in
    numpy at N = 32768 on the reference generator's inputs) decides the iteration count with
    margin: the step before convergence is >= 10x above tol and the converged step >= 4x below,
    so summation-order rounding (~1e-16 relative per entry) cannot move the count."""
    g = golden("config3_trace.npz")
    assert int(g["n"]) == 32768 and float(g["tol"]) == 1e-12
    it = int(g["iterations_rel_fro"])
    steps = np.asarray(g["steps"])
    assert steps[it - 1] <= 1e-12 < steps[it - 2]
    assert steps[it - 2] >= 10 * 1e-12 and steps[it - 1] <= 0.25e-12
    itm = int(g["iterations_max_abs"])
    mx = np.asarray(g["max_abs"])
    assert mx[itm - 1] < 1e-12 <= mx[itm - 2]
    assert np.all(np.diff(np.log10(steps)) < -1.5)  # monotone, geometric convergence
