"""Randomised parity cases against the reference build (oracle/_ref, the unmodified
reference compiled from its sources): shared by tests/test_gpu_fuzz_parity.py (a fixed
seeded subset) and tools/parity_sweep.py (a long sweep whose summary is committed under
profiles/). Each case draws an entry point, a size from the edge set the reference's own
tests use (1, 2, 3, 5, 7, 8, 16, 33, 64, ... and tile / row-group boundaries), real or
complex values, dense or CSR storage, a coupling and a seed, runs the device path through
the public Python API and the reference on the same inputs, and checks north_star's
tolerances: eigenvalues 1e-10 relative, eigenvectors 1e-9, iterations +-1, same status."""
import numpy as np

import paper_2012_14702_b200 as ipt

import os

SIZES = [1, 2, 3, 5, 7, 8, 15, 16, 17, 31, 33, 63, 64, 65, 127, 128, 129, 200, 255, 256, 257, 300, 511, 513]
if os.environ.get("PARITY_BIG") == "1":  # several K1 / INT8 tiles, ragged (slow on the CPU reference)
    SIZES = [700, 1000, 1023, 1100, 1500]
KINDS = ["full", "full_csr", "single", "single_csr", "continuation", "accelerated", "apply_map_full",
         "matmul", "matvec", "matvec_csr"]


def _matrix(rng, n, cplx, csr, eps):
    gaps = rng.uniform(0.6, 1.6, n)
    d = np.cumsum(gaps) + rng.uniform(-0.2, 0.2)
    if cplx:
        d = d + 1j * rng.uniform(-0.3, 0.3, n)
    if csr:
        density = min(1.0, rng.uniform(2.0, 12.0) / max(n, 1))
        mask = rng.random((n, n)) < density
    else:
        mask = np.ones((n, n), bool)
    np.fill_diagonal(mask, False)
    vals = rng.uniform(-1.0, 1.0, (n, n))
    if cplx:
        vals = vals + 1j * rng.uniform(-1.0, 1.0, (n, n))
    delta = np.where(mask, eps * vals, 0.0)
    if csr:
        r, c = np.nonzero(delta)
        return d, ipt.CsrMatrix.from_triplets(n, n, r, c, delta[r, c]), delta
    return d, delta, delta


def draw(case_seed):
    rng = np.random.default_rng(case_seed)
    kind = KINDS[rng.integers(len(KINDS))]
    n = int(SIZES[rng.integers(len(SIZES))])
    cplx = bool(rng.random() < 0.35) and kind != "accelerated"
    csr = kind.endswith("csr")
    eps = float(rng.uniform(0.02, 0.5) / np.sqrt(max(n, 1)))
    return rng, kind, n, cplx, csr, eps


def run_case(case_seed, ref):
    """One case: returns (kind, n, cplx, max eigenvector diff, max eigenvalue rel diff, note);
    raises AssertionError on a parity failure."""
    rng, kind, n, cplx, csr, eps = draw(case_seed)
    d, delta, dense = _matrix(rng, n, cplx, csr or kind == "matvec_csr", eps)
    p = ipt.Partition(d, delta)
    tol = 1e-12
    cfg = ipt.IterationConfig(tolerance=tol)
    dz = dl = 0.0
    if kind in ("full", "full_csr"):
        r = ipt.solve_full(p, ipt.build_gaps(p), cfg)
        o = ref.solve_full_csr(d, delta, tol=tol) if csr else ref.solve_full(d, delta, tol=tol)
        assert r.status.value == o["status"], (r.status, o["status"])
        if o["status"] == 0:
            assert abs(r.iterations - o["iterations"]) <= 1, (r.iterations, o["iterations"])
            dz = float(np.max(np.abs(r.Z - o["Z"])))
            lam = o["eigenvalues"]
            dl = float(np.max(np.abs(r.eigenvalues - lam) / np.maximum(np.abs(lam), 1e-300)))
            assert dz <= 1e-9 and dl <= 1e-10, (dz, dl)
    elif kind in ("single", "single_csr", "continuation", "accelerated"):
        a = int(rng.integers(n))
        g = ipt.build_gaps(p)
        if kind == "continuation":
            r = ipt.solve_single_continuation(p, g, a, cfg, 0.6)
            o = ref.solve_single(d, delta, a, tol=tol, mode="continuation", alpha=0.6)
        elif kind == "accelerated":
            c2 = ipt.IterationConfig(tolerance=tol, residual_tolerance=1e-11)
            r = ipt.solve_single_accelerated(p, g, a, c2, memory=3)
            o = ref.solve_single(d, delta, a, tol=tol, mode="accelerated", memory=3, residual_tol=1e-11)
        else:
            r = ipt.solve_single(p, g, a, cfg)
            o = ref.solve_single(d, delta, a, tol=tol)
        assert r.status.value == o["status"], (r.status, o["status"])
        if o["status"] == 0:
            assert abs(r.iterations - o["iterations"]) <= (2 if kind == "accelerated" else 1), \
                (r.iterations, o["iterations"])
            dz = float(np.max(np.abs(r.z - o["z"])))
            dl = float(abs(r.eigenvalue - o["eigenvalue"]) / max(abs(o["eigenvalue"]), 1e-300))
            assert dz <= 1e-9 and dl <= 1e-10, (dz, dl)
    elif kind == "apply_map_full":
        z = np.eye(n) + 0.01 * rng.standard_normal((n, n)) * (1 + (1j if cplx else 0))
        np.fill_diagonal(z, 1.0)
        f = ipt.apply_map_full(p, ipt.build_gaps(p), z)
        o = ref.apply_map_full(d, delta, z)
        dz = float(np.max(np.abs(f - o)))
        assert dz <= 1e-12 * max(1.0, float(np.max(np.abs(o)))), dz
    elif kind == "matmul":
        b = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
        c = ipt.kernels.matmul(dense, b)
        o = ref.matmul(dense, b)
        scale = max(1e-300, float(np.linalg.norm(dense) * np.linalg.norm(b)))
        dz = float(np.max(np.abs(c - o)))
        assert dz <= 1e-13 * scale, (dz, scale)  # test_kernels.cpp:40-50
    else:  # matvec / matvec_csr
        x = rng.standard_normal(n) + (1j * rng.standard_normal(n) if cplx else 0)
        y = ipt.kernels.matvec(delta, x)
        o = ref.matvec(delta, x)
        dz = float(np.max(np.abs(y - o)))
        assert dz <= 1e-13 * max(1.0, float(np.max(np.abs(o)))), dz
    return kind, n, cplx, dz, dl


# ---- extended cases: warm starts, the max-abs stop rule, the Ozaki product, in-process
# ranks, non-convergent couplings (Diverged / MaxIterations parity) and traces
KINDS_EXT = ["full_warm", "single_warm", "full_maxabs", "full_ozaki", "full_ranks", "single_ranks_csr",
             "full_hard", "single_hard"]


def draw_ext(case_seed):
    rng = np.random.default_rng(case_seed)
    kind = KINDS_EXT[rng.integers(len(KINDS_EXT))]
    n = int(SIZES[rng.integers(len(SIZES))])
    cplx = bool(rng.random() < 0.35) and kind not in ("full_ozaki", "single_ranks_csr")
    eps = float(rng.uniform(0.02, 0.5) / np.sqrt(max(n, 1)))
    if kind.endswith("hard"):
        eps = float(rng.uniform(0.3, 3.0))  # gaps ~1: divergence or slow convergence
    return rng, kind, n, cplx, eps


STATUS_COUNTS = {0: 0, 1: 0, 2: 0}  # reference statuses met by the extended cases (sweep summary)


def _compare_full(r, o, trace=False):
    assert r.status.value == o["status"], (r.status, o["status"])
    STATUS_COUNTS[o["status"]] += 1
    if o["status"] != 0:
        assert abs(r.iterations - o["iterations"]) <= 1, (r.iterations, o["iterations"])
        return 0.0, 0.0
    assert abs(r.iterations - o["iterations"]) <= 1, (r.iterations, o["iterations"])
    dz = float(np.max(np.abs(r.Z - o["Z"])))
    lam = o["eigenvalues"]
    dl = float(np.max(np.abs(r.eigenvalues - lam) / np.maximum(np.abs(lam), 1e-300)))
    assert dz <= 1e-9 and dl <= 1e-10, (dz, dl)
    if trace and r.iterations == o["iterations"]:
        tr = np.asarray(r.trace)
        assert np.allclose(tr, o["trace"], rtol=1e-6, atol=1e-15), (tr, o["trace"])
    return dz, dl


def _compare_single(r, o):
    assert r.status.value == o["status"], (r.status, o["status"])
    STATUS_COUNTS[o["status"]] += 1
    assert abs(r.iterations - o["iterations"]) <= 1, (r.iterations, o["iterations"])
    if o["status"] != 0:
        return 0.0, 0.0
    dz = float(np.max(np.abs(r.z - o["z"])))
    dl = float(abs(r.eigenvalue - o["eigenvalue"]) / max(abs(o["eigenvalue"]), 1e-300))
    assert dz <= 1e-9 and dl <= 1e-10, (dz, dl)
    return dz, dl


def run_case_ext(case_seed, ref):
    from paper_2012_14702_b200 import dist

    rng, kind, n, cplx, eps = draw_ext(case_seed)
    csr = kind.endswith("csr")
    d, delta, dense = _matrix(rng, n, cplx, csr, eps)
    p = ipt.Partition(d, delta)
    g = ipt.build_gaps(p)
    tol = 1e-12
    cfg = ipt.IterationConfig(tolerance=tol, max_iterations=60, record_trace=True)
    if kind == "full_warm":
        w = np.eye(n) + 0.05 * eps * rng.standard_normal((n, n))
        w = w.astype(complex) if cplx else w
        np.fill_diagonal(w, 1.0 + (0.3j if cplx else 0.0))
        r = ipt.solve_full(p, g, cfg, warm_start=w)
        o = ref.solve_full(d, delta, tol=tol, max_iter=60, record_trace=True, warm=w)
        dz, dl = _compare_full(r, o, trace=True)
    elif kind == "single_warm":
        a = int(rng.integers(n))
        w = 0.01 * rng.standard_normal(n) + (0.01j * rng.standard_normal(n) if cplx else 0)
        w[a] = 1.0 + (0.5j if cplx else 0.0)
        r = ipt.solve_single(p, g, a, cfg, warm_start=w)
        o = ref.solve_single(d, delta, a, tol=tol, max_iter=60, warm=w)
        dz, dl = _compare_single(r, o)
    elif kind == "full_maxabs":
        c2 = ipt.IterationConfig(tolerance=tol, max_iterations=60, stop_rule="max_abs")
        r = ipt.solve_full(p, g, c2)
        o = ref.solve_full(d, delta, tol=tol, max_iter=60, stop_rule="max_abs")
        dz, dl = _compare_full(r, o)
    elif kind == "full_ozaki":
        r = ipt.solve_full(p, g, cfg, product="ozaki")
        o = ref.solve_full(d, delta, tol=tol, max_iter=60, record_trace=True)
        dz, dl = _compare_full(r, o, trace=True)
    elif kind == "full_ranks":
        k = int(rng.integers(2, 4))
        ctxs = dist.local_contexts(k)
        try:
            r = dist.run_ranks(lambda c: ipt.solve_full(p, g, cfg, ctx=c), ctxs)[0]
        finally:
            for c in ctxs:
                c.close()
        o = ref.solve_full(d, delta, tol=tol, max_iter=60, record_trace=True)
        dz, dl = _compare_full(r, o, trace=True)
    elif kind == "single_ranks_csr":
        k = int(rng.integers(2, 4))
        a = int(rng.integers(n))
        ctxs = dist.local_contexts(k)
        try:
            r = dist.run_ranks(lambda c: ipt.solve_single(p, g, a, cfg, ctx=c), ctxs)[0]
        finally:
            for c in ctxs:
                c.close()
        o = ref.solve_single(d, delta, a, tol=tol, max_iter=60)
        dz, dl = _compare_single(r, o)
    elif kind == "full_hard":
        r = ipt.solve_full(p, g, cfg)
        o = ref.solve_full(d, delta, tol=tol, max_iter=60, record_trace=True)
        dz, dl = _compare_full(r, o)
    else:  # single_hard
        a = int(rng.integers(n))
        r = ipt.solve_single(p, g, a, cfg)
        o = ref.solve_single(d, delta, a, tol=tol, max_iter=60)
        dz, dl = _compare_single(r, o)
    return kind, n, cplx, dz, dl


# ---- the C++ drop-in layer (tests/cpp/cpp_api_shim.cpp): the reference's own entry points
# on ComplexMatrix carriers, against the Python mirror (the same device path: bitwise) and
# the reference build (north_star tolerances); with several in-process ranks
# (ipt::b200::set_devices) and repeated solve_single calls (device-resident problem)
KINDS_CPP = ["cpp_full", "cpp_full_csr", "cpp_single", "cpp_single_csr", "cpp_continuation", "cpp_matvec",
             "cpp_matmul", "cpp_full_devices", "cpp_single_repeat"]
_SHIM = None


def shim():
    global _SHIM
    if _SHIM is None:
        import ctypes as C

        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2012_14702_b200",
                            "_build", "libcpp_api_shim.so")
        _SHIM = C.CDLL(path)
        _SHIM.shim_last_error.restype = C.c_char_p
    return _SHIM


def _ic(a):
    """interleaved complex128 view (C-contiguous)"""
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def draw_cpp(case_seed):
    rng = np.random.default_rng(case_seed)
    kind = KINDS_CPP[rng.integers(len(KINDS_CPP))]
    n = int(SIZES[rng.integers(len(SIZES))])
    cplx = bool(rng.random() < 0.35)
    eps = float(rng.uniform(0.02, 0.5) / np.sqrt(max(n, 1)))
    return rng, kind, n, cplx, eps


def run_case_cpp(case_seed, ref):
    import ctypes as C

    rng, kind, n, cplx, eps = draw_cpp(case_seed)
    csr = kind.endswith("csr") or kind == "cpp_matvec" and rng.random() < 0.5
    d, delta_obj, dense = _matrix(rng, n, cplx, csr, eps)
    L = shim()
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    dc, ac = _ic(d), _ic(dense)
    tol = 1e-12
    stats = np.zeros(5)

    def chk(rc):
        if rc != 0:
            raise RuntimeError(L.shim_last_error().decode())

    p = ipt.Partition(d, delta_obj)
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=tol)
    dz = dl = 0.0
    if kind in ("cpp_full", "cpp_full_csr", "cpp_full_devices"):
        devs = np.zeros(int(rng.integers(2, 4)) if kind == "cpp_full_devices" else 0, dtype=np.int32)
        z = np.empty((n, n), np.complex128)
        lam = np.empty(n, np.complex128)
        chk(L.shim_solve_full(C.c_int64(n), P(dc), P(ac), C.c_int(1 if csr else 0), C.c_double(tol), C.c_int(1000),
                              C.c_int(devs.size), P(devs), P(z), P(lam), P(stats)))
        r = ipt.solve_full(p, g, cfg)
        assert int(stats[0]) == r.iterations and int(stats[1]) == r.status.value
        assert np.array_equal(z, r.Z.astype(np.complex128)), np.max(np.abs(z - r.Z))  # same device path
        assert np.array_equal(lam, np.asarray(r.eigenvalues, dtype=np.complex128))
        o = ref.solve_full_csr(d, delta_obj, tol=tol) if csr else ref.solve_full(d, dense, tol=tol)
        if o["status"] == 0:
            assert abs(int(stats[0]) - o["iterations"]) <= 1
            dz = float(np.max(np.abs(z - o["Z"])))
            dl = float(np.max(np.abs(lam - o["eigenvalues"]) / np.maximum(np.abs(o["eigenvalues"]), 1e-300)))
            assert dz <= 1e-9 and dl <= 1e-10, (dz, dl)
    elif kind in ("cpp_single", "cpp_single_csr", "cpp_continuation", "cpp_single_repeat"):
        a = int(rng.integers(n))
        mode = 1 if kind == "cpp_continuation" else 0
        repeat = 3 if kind == "cpp_single_repeat" else 1
        z = np.empty(n, np.complex128)
        lam = np.empty(1, np.complex128)
        chk(L.shim_solve_single(C.c_int64(n), P(dc), P(ac), C.c_int(1 if csr else 0), C.c_int64(a),
                                C.c_double(tol), C.c_int(1000), C.c_int(mode), C.c_double(0.6), C.c_int(repeat),
                                C.c_int(0), None, P(z), P(lam), P(stats)))
        r = (ipt.solve_single_continuation(p, g, a, cfg, 0.6) if mode else ipt.solve_single(p, g, a, cfg))
        assert int(stats[0]) == r.iterations and int(stats[1]) == r.status.value
        assert np.array_equal(z, np.asarray(r.z, dtype=np.complex128)), np.max(np.abs(z - r.z))
        o = (ref.solve_single(d, delta_obj, a, tol=tol, mode="continuation", alpha=0.6) if mode
             else ref.solve_single(d, delta_obj, a, tol=tol))
        if o["status"] == 0:
            assert abs(int(stats[0]) - o["iterations"]) <= 1
            dz = float(np.max(np.abs(z - o["z"])))
            dl = float(abs(lam[0] - o["eigenvalue"]) / max(abs(o["eigenvalue"]), 1e-300))
            assert dz <= 1e-9 and dl <= 1e-10, (dz, dl)
    elif kind == "cpp_matvec":
        x = _ic(rng.standard_normal(n) + (1j * rng.standard_normal(n) if cplx else 0))
        y = np.empty(n, np.complex128)
        chk(L.shim_matvec(C.c_int64(n), P(ac), C.c_int(1 if csr else 0), P(x), P(y)))
        o = ref.matvec(dense, x)
        dz = float(np.max(np.abs(y - o), initial=0.0))
        assert dz <= 1e-13 * max(1.0, float(np.max(np.abs(o), initial=0.0))), dz
    else:  # cpp_matmul
        b = _ic(rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0))
        c = np.empty((n, n), np.complex128)
        chk(L.shim_matmul(C.c_int64(n), P(ac), P(b), P(c)))
        o = ref.matmul(dense, b)
        scale = max(1e-300, float(np.linalg.norm(dense) * np.linalg.norm(b)))
        dz = float(np.max(np.abs(c - o)))
        assert dz <= 1e-13 * scale, (dz, scale)
    return kind, n, cplx, dz, dl
