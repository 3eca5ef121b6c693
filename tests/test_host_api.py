"""Host-side logic of the drop-in API (CPU only): partition / gaps / CSR rules,
synthetic configurations, and that the C ABI library loads and exports every
symbol the headers declare (no compute calls without a GPU)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import _lib, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ipt_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header", ["ipt_cuda.h", "ipt_synth.h"])
def test_library_exports_every_declared_symbol(header):
    lib = C.CDLL(_lib.LIB_PATH)
    names = declared_functions(header)
    assert len(names) >= 5
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes binding covers them with a signature
    assert not [n for n in names if n not in _lib.SIGNATURES]


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_default_params_match_iteration_config():
    p = _lib.default_params()
    cfg = ipt.IterationConfig()
    assert p.tolerance == cfg.tolerance == 100 * np.finfo(float).eps
    assert p.max_iterations == cfg.max_iterations == 1000
    assert p.divergence_threshold == cfg.divergence_threshold == 1e8


def test_partition_dense_and_csr():
    m = np.array([[1.0, 2.0, 0.0], [3.0, 4.0, 5.0], [0.0, 6.0, 7.0]])
    p = ipt.partition(m)
    assert np.array_equal(p.d, [1, 4, 7])
    assert np.array_equal(np.diag(p.delta), [0, 0, 0])
    assert np.array_equal(ipt.reconstruct(p), m)
    rows, cols = np.nonzero(m)
    s = ipt.CsrMatrix.from_triplets(3, 3, rows, cols, m[rows, cols])
    ps = ipt.partition(s)
    assert np.array_equal(ps.d, [1, 4, 7])
    assert np.array_equal(ps.delta.to_dense(), p.delta)


def test_csr_rejects_duplicates_and_drops_zeros():
    """complex_matrix.cpp:39-69."""
    with pytest.raises(ValueError):
        ipt.CsrMatrix.from_triplets(2, 2, [0, 0], [1, 1], [1.0, 2.0])
    with pytest.raises(ValueError):
        ipt.CsrMatrix.from_triplets(2, 2, [0], [2], [1.0])
    s = ipt.CsrMatrix.from_triplets(2, 2, [1, 0, 0], [0, 1, 0], [3.0, 0.0, 5.0])
    assert s.nnz == 2 and list(s.col_indices) == [0, 0] and list(s.row_offsets) == [0, 1, 2]


def test_build_gaps_degeneracy(ref_arm):
    """partition.cpp:54-94: default tolerance 1e-12 max|d|, sweep over real-sorted d."""
    p = ipt.Partition(np.array([0.0, 1.0, 1.0 + 1e-13]), np.zeros((3, 3)))
    with pytest.raises(ipt.DegenerateDiagonal) as e:
        ipt.build_gaps(p)
    assert (e.value.i, e.value.j) == (1, 2)
    ipt.build_gaps(p, 0.0)  # explicit zero tolerance accepts distinct entries
    g = ipt.build_gaps(ipt.Partition(np.array([0.0, 1.0, 3.0]), np.zeros((3, 3))))
    assert g.entry(0, 1) == -1.0 and g.entry(1, 1) == 0.0
    assert np.allclose(g.column(0), [0.0, 1.0, 1.0 / 3.0])


def test_build_gaps_agrees_with_reference_on_config5_pattern(ref_arm):
    p = synth.csr_ci(1 << 16)
    import ctypes

    ij = np.zeros(2, dtype=np.int64)
    rc_ref = ref_arm.lib.ref_build_gaps(ctypes.c_int64(p.size()), np.ascontiguousarray(p.d, np.complex128).ctypes.data_as(
        ctypes.POINTER(ctypes.c_double)), ctypes.c_double(-1.0), ij.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    try:
        ipt.build_gaps(p)
        ours = 0
    except ipt.DegenerateDiagonal as e:
        ours = -3
        assert (e.i, e.j) == tuple(ij)
    assert ours == rc_ref


def test_config_generators_structure():
    p = synth.dense_uniform(64, 0.01)
    assert np.array_equal(p.d, np.arange(1, 65))
    assert np.array_equal(p.delta, p.delta.T) and np.all(np.diag(p.delta) == 0)
    assert np.max(np.abs(p.delta)) <= 0.01
    q = synth.dense_normal(200)
    assert np.array_equal(q.delta, q.delta.T) and np.all(np.diag(q.delta) == 0)
    assert np.all(np.diff(q.d) >= 1.0)  # gaps >= 1 by construction
    c = synth.csr_ci(4096, 32)
    dense = c.delta.to_dense()
    assert np.array_equal(dense, dense.T) and np.all(np.diag(dense) == 0)
    assert np.all(np.diff(c.d) >= 0)
    for i in range(0, 4096, 97):  # sorted, duplicate-free rows
        cols = c.delta.col_indices[c.delta.row_offsets[i]:c.delta.row_offsets[i + 1]]
        assert np.all(np.diff(cols) > 0)
    assert 32 * 4096 <= c.delta.nnz <= 64 * 4096


def test_invalid_config_is_rejected_before_any_device_call():
    p = ipt.Partition(np.array([0.0, 1.0]), np.zeros((2, 2)))
    with pytest.raises(ValueError):
        ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=-1.0))
    with pytest.raises(ValueError):
        ipt.solve_single(p, ipt.build_gaps(p), 5)
    with pytest.raises(ValueError):
        ipt.solve_single_continuation(p, ipt.build_gaps(p), 0, shrink_alpha=1.5)


def test_devices_argument_is_validated_before_any_device_call():
    p = ipt.Partition(np.array([0.0, 1.0]), np.zeros((2, 2)))
    g = ipt.build_gaps(p)
    fake_ctx = object()
    with pytest.raises(ValueError):
        ipt.solve_full(p, g, devices=[0, 1], ctx=fake_ctx)
    with pytest.raises(ValueError):
        ipt.solve_full(p, g, devices=[0, 1], out=(None, None, None, None))
    with pytest.raises(ValueError):
        ipt.solve_single(p, g, 0, devices=[0, 1], ctx=fake_ctx)


def test_product_does_not_import_oracle():
    """The product path must never route through the CPU oracle."""
    pkg = os.path.join(ROOT, "paper_2012_14702_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in src and "libipt_oracle" not in src and "libipt_ref" not in src, f
