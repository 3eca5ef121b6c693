"""Generate the golden fixtures under tests/golden/ from the REFERENCE build.

Runs here (where /root/reference exists) against oracle/_ref/libipt_ref.so,
i.e. the unmodified reference sources compiled by oracle/Makefile. The GPU box
never runs this script; it only reads the committed .npz files.

    python tests/golden/make_golden.py            # small + config 1 + config 4/5 at reduced size
    python tests/golden/make_golden.py --big      # + config 2/3 column samples, config 5 full size

Each fixture records the reference entry point it came from.
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
EPS = np.finfo(float).eps


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


def explicit_2x2(eps):  # proj/src/testgen.cpp:196-201
    return np.array([0.0, 1.0]), np.array([[0.0, eps], [eps, 0.0]], dtype=complex)


def explicit_3x3(eps):  # proj/src/testgen.cpp:203-210
    e = complex(eps)
    return np.array([0.0, 1.0, 3.0]), e * np.array([[0, 1, 2], [1, 0, 3], [2, 3, 0]], dtype=complex)


def split(m):
    d = np.diag(m).copy()
    delta = m.copy()
    np.fill_diagonal(delta, 0)
    return d, delta


def random_dense_ref(n, seed):
    """test_solver.cpp:15-20: cplx(rng.normal(), rng.normal()) row-major from Rng(seed)."""
    v = oracle.ref().rng_draws(seed, 2, 2 * n * n)
    return (v[0::2] + 1j * v[1::2]).reshape(n, n)


def small_cases():
    R = oracle.ref()
    out = {}
    # test_solver.cpp:24-32, :65-75, :126-133, :181-187, :210-214, :218-227
    for eps in (0.05, 0.1, 0.3, 1.0, 3.0):
        d, delta = explicit_2x2(eps)
        s = R.solve_single(d, delta, 0, record_trace=True)
        f = R.solve_full(d, delta, record_trace=True)
        out[f"x2_{eps}_single_z"] = s["z"]
        out[f"x2_{eps}_single_meta"] = np.array([s["iterations"], s["status"], s["residual"], s["final_step"],
                                                 s["matvec_count"], s["eigenvalue"].real, s["eigenvalue"].imag])
        out[f"x2_{eps}_full_Z"] = f["Z"]
        out[f"x2_{eps}_full_lam"] = f["eigenvalues"]
        out[f"x2_{eps}_full_meta"] = np.array([f["iterations"], f["status"], f["residual_frobenius"],
                                               f["sigma_min"], f["final_step"], f["matmul_count"]])
        out[f"x2_{eps}_map1"] = R.apply_map_full(d, delta, np.eye(2))
        c = R.solve_single(d, delta, 0, mode="continuation", alpha=0.0)
        out[f"x2_{eps}_cont0_meta"] = np.array([c["iterations"], c["status"], c["eigenvalue"].real])
        out[f"x2_{eps}_cont0_z"] = c["z"]
    # 3x3: test_testgen.cpp:138-147 and the pinned continuation point (fixtures.hpp:13)
    d, delta = explicit_3x3(0.05)
    f = R.solve_full(d, delta)
    out["x3_0.05_full_lam"] = f["eigenvalues"]
    out["x3_0.05_full_Z"] = f["Z"]
    out["x3_0.05_map_single"] = R.apply_map_single(d, delta, 0, np.array([1, 0, 0], dtype=complex))
    d, delta = explicit_3x3(-0.475)
    p = R.solve_single(d, delta, 1, max_iter=4000)
    c = R.solve_single(d, delta, 1, max_iter=4000, mode="continuation", alpha=0.9)
    out["x3_pinned_plain_meta"] = np.array([p["iterations"], p["status"]])
    out["x3_pinned_cont_meta"] = np.array([c["iterations"], c["status"], c["residual"]])
    out["x3_pinned_cont_z"] = c["z"]
    # gen_near_diagonal cases of test_solver.cpp:158-209 (dense, normal R, not symmetric)
    for (n, eps, seed) in ((8, 0.01, 2024), (10, 0.02, 7), (16, 0.002, 8), (256, 0.02, 9000)):
        m = R.gen_near_diagonal(n, eps, False, seed)
        d, delta = split(m)
        f = R.solve_full(d, delta, record_trace=True)
        key = f"nd_{n}_{seed}"
        out[key + "_M"] = m
        out[key + "_Z"] = f["Z"]
        out[key + "_lam"] = f["eigenvalues"]
        out[key + "_trace"] = f["trace"]
        out[key + "_meta"] = np.array([f["iterations"], f["status"], f["residual_frobenius"], f["sigma_min"],
                                       f["final_step"], f["matmul_count"]])
        if n <= 16:
            out[key + "_direct"] = R.dense_eigenvalues(m)
        for j in (0, n // 2, n - 1):
            s = R.solve_single(d, delta, j)
            out[key + f"_single{j}_z"] = s["z"]
            out[key + f"_single{j}_meta"] = np.array([s["iterations"], s["status"], s["eigenvalue"].real,
                                                      s["eigenvalue"].imag, s["residual"]])
    # complex random cases (test_solver.cpp:134-154): map columns vs single map
    m = random_dense_ref(6, 41)
    d, delta = split(m)
    z = random_dense_ref(6, 42)
    np.fill_diagonal(z, 1.0)
    out["cx6_M"] = m
    out["cx6_Zin"] = z
    out["cx6_F"] = R.apply_map_full(d, delta, z)
    out["cx6_single"] = np.stack([R.apply_map_single(d, delta, j, z[:, j]) for j in range(6)], axis=1)
    # kernels: matmul / matvec on complex inputs (test_kernels.cpp:40-50)
    for n in (1, 2, 3, 7, 16, 33, 64):
        a = random_dense_ref(n, 10 + n)
        b = random_dense_ref(n, 20 + n)
        out[f"mm_{n}_A"] = a
        out[f"mm_{n}_B"] = b
        out[f"mm_{n}_C"] = R.matmul(a, b)
    # certified complex family of acceptance #2 at a few sizes (complex d, complex Delta)
    save("small_cases.npz", **out)


def config1():
    R = oracle.ref()
    p = synth.config1()
    out = dict(d=p.d)
    cols = np.array([0, 1, 341, 512, 1022, 1023])
    for rule, tol in (("rel_fro", 1e-12), ("max_abs", 1e-12), ("rel_fro", 100 * EPS)):
        t0 = time.time()
        r = R.solve_full(p.d, p.delta, tol=tol, stop_rule=rule, record_trace=True)
        tag = f"{rule}_{'default' if tol < 1e-13 else 'tol12'}"
        out[tag + "_lam"] = r["eigenvalues"].real
        out[tag + "_cols"] = r["Z"][:, cols].real
        out[tag + "_trace"] = r["trace"]
        out[tag + "_meta"] = np.array([r["iterations"], r["status"], r["residual_frobenius"], r["sigma_min"],
                                       r["final_step"], r["final_max_abs"], r["matmul_count"]])
        out[tag + "_zsum"] = np.array([r["Z"].real.sum(), np.abs(r["Z"].real).sum()])
        print(f"config1 {tag}: {r['iterations']} it, {time.time() - t0:.1f}s", flush=True)
    out["cols"] = cols
    save("config1.npz", **out)


def single_configs(big):
    R = oracle.ref()
    out = {}
    # config 4 construction at reduced size (dense GEMV path)
    for n in ([4096, 32768] if big else [4096]):
        p = synth.dense_normal(n)
        s = R.solve_single(p.d, p.delta, 0, tol=1e-12, record_trace=True)
        out[f"c4_{n}_z"] = s["z"].real
        out[f"c4_{n}_meta"] = np.array([s["iterations"], s["status"], s["eigenvalue"].real, s["residual"],
                                        s["final_step"], s["matvec_count"]])
        out[f"c4_{n}_trace"] = s["trace"]
        print(f"config4 n={n}: {s['iterations']} it, lambda0={s['eigenvalue'].real!r}", flush=True)
    # config 5 construction at reduced and (big) full size (CSR SpMV path)
    for n in ([1 << 16, 1 << 21] if big else [1 << 16]):
        p = synth.csr_ci(n)
        s = R.solve_single(p.d, p.delta, 0, tol=1e-10, degeneracy_tol=0.0, record_trace=True)
        key = f"c5_{n}"
        if n <= (1 << 16):
            out[key + "_z"] = s["z"].real
        else:
            idx = np.argsort(-np.abs(s["z"].real))[:64]
            out[key + "_zidx"] = idx
            out[key + "_zval"] = s["z"].real[idx]
            out[key + "_znorm"] = np.array([np.linalg.norm(s["z"])])
        out[key + "_meta"] = np.array([s["iterations"], s["status"], s["eigenvalue"].real, s["residual"],
                                       s["final_step"], s["matvec_count"], p.delta.nnz])
        out[key + "_trace"] = s["trace"]
        print(f"config5 n={n}: nnz={p.delta.nnz} {s['iterations']} it lambda0={s['eigenvalue'].real!r}", flush=True)
    save("single_configs.npz", **out)


def accelerated():
    """solve_single_accelerated (anderson.cpp:184-247) on the acceptance #7 instance
    (gen_fci_like N=4096, density 50/N, gap 20, seed 2718281828) and two variants."""
    R = oracle.ref()
    out = {}
    for name, (n, dens, gap, seed) in {"acc7": (4096, 50.0 / 4096, 20.0, 2718281828),
                                       "fci2k": (2048, 40.0 / 2048, 5.0, 77)}.items():
        d, delta = R.gen_fci_like(n, dens, gap, seed)
        out[name + "_d"] = d
        out[name + "_rowptr"] = delta.row_offsets
        out[name + "_cols"] = delta.col_indices
        out[name + "_vals"] = delta.values
        for mem in (0, 2, 5):
            a = R.solve_single(d, delta, 0, mode="accelerated", memory=mem, residual_tol=1e-8, record_trace=True)
            key = f"{name}_m{mem}"
            out[key + "_z"] = a["z"].real
            out[key + "_meta"] = np.array([a["iterations"], a["status"], a["eigenvalue"].real, a["residual"],
                                           a["final_step"], a["matvec_count"]])
            out[key + "_trace"] = a["trace"]
            print(f"{key}: {a['matvec_count']} matvecs, status {a['status']}", flush=True)
        p = R.solve_single(d, delta, 0, residual_tol=1e-8)
        out[name + "_plain_meta"] = np.array([p["iterations"], p["status"], p["eigenvalue"].real, p["matvec_count"]])
    save("accelerated.npz", **out)


def full_columns(big):
    """Configs 2/3: reference solve_single(j) columns (test_solver.cpp:188-201 route)."""
    R = oracle.ref()
    out = {}
    for n in ([8192, 32768] if big else [8192]):
        p = synth.config3(n=n)
        rng = np.random.default_rng(n)
        cols = np.unique(np.concatenate([[0, 1, n // 2, n - 2, n - 1], rng.integers(0, n, 11)]))  # >= 16
        out[f"n{n}_cols"] = cols
        z, its, status, lam = R.solve_single_multi(p.d, p.delta, cols, tol=1e-12)
        del p
        out[f"n{n}_z"] = z.real
        out[f"n{n}_lam"] = lam.real
        out[f"n{n}_its"] = its
        print(f"full columns n={n}: lam0={out[f'n{n}_lam'][0]!r}", flush=True)
    save("full_columns.npz", **out)


def sparse_full():
    """solve_full / apply_map_full on CSR partitions: the reference's sparse product
    path (kernels.cpp:88-108) on gen_fci_like instances (testgen.cpp:174-194), and the
    config 5 CI-like construction at N=4096 (diverges: meta only)."""
    R = oracle.ref()
    out = {}
    for name, (n, dens, gap, seed) in {"f256": (256, 16 / 256, 20.0, 11),
                                       "f1024": (1024, 24 / 1024, 20.0, 12)}.items():
        d, delta = R.gen_fci_like(n, dens, gap, seed)
        out[name + "_d"] = d
        out[name + "_rowptr"] = delta.row_offsets
        out[name + "_cols"] = delta.col_indices
        out[name + "_vals"] = delta.values
        r = R.solve_full_csr(d, delta)
        if n <= 256:
            out[name + "_Z"] = r["Z"].real
            z0 = np.random.default_rng(seed).standard_normal((n, n))
            np.fill_diagonal(z0, 1.0)
            out[name + "_map_in"] = z0
            out[name + "_map_out"] = R.apply_map_full_csr(d, delta, z0).real
        else:
            cols = np.array([0, 1, n // 2, n - 1])
            out[name + "_zcols_idx"] = cols
            out[name + "_zcols"] = r["Z"].real[:, cols]
        out[name + "_lam"] = r["eigenvalues"].real
        out[name + "_meta"] = np.array([r["iterations"], r["status"], r["final_step"], r["residual_frobenius"],
                                        r["sigma_min"], r["matmul_count"]])
        print(f"sparse full {name}: nnz={delta.nnz} {r['iterations']} it status {r['status']}", flush=True)
    p = synth.csr_ci(4096)
    r = R.solve_full_csr(p.d, p.delta, tol=1e-10)
    out["ci4096_meta"] = np.array([r["iterations"], r["status"], p.delta.nnz])
    print(f"sparse full ci4096: {r['iterations']} it status {r['status']}", flush=True)
    save("sparse_full.npz", **out)


def lu_case():
    """lu_factor / lu_solve_matrix (lu.cpp:10-103) on a seeded complex 96 x 96 matrix."""
    R = oracle.ref()
    rng = np.random.default_rng(2024)
    a = rng.standard_normal((96, 96)) + 1j * rng.standard_normal((96, 96))
    b = rng.standard_normal((96, 5)) + 1j * rng.standard_normal((96, 5))
    lu, perm, sing = R.lu_factor(a)
    x = R.lu_solve(a, b)
    save("lu.npz", a=a, lu=lu, perm=perm, b=b, x=x, singular=np.array([sing]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    oracle.build()
    jobs = dict(small=small_cases, config1=config1, accel=accelerated, single=lambda: single_configs(a.big),
                columns=lambda: full_columns(a.big), sparse=sparse_full, lu=lu_case)
    for name, fn in jobs.items():
        if a.only and name not in a.only.split(","):
            continue
        fn()
