"""The CSR map's kernels give the same bits: the default (spmv_pipe_kernel: folded row
sums, software-pipelined loads, variant 30), the folded-sum kernel (20) and the round-1/2
group kernel (16) form every row sum over the same lanes in the same order, so iterates,
eigenvalues, stop sums and the plain matvec agree bit for bit (ipt_single.cu). Each variant
runs in its own process (IPT_SPMV_VARIANT is read once)."""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import synth

def ragged(n, seed):
    # empty rows, one-entry rows, rows longer than one chunk (64 and 128 entries per pass),
    # n not a multiple of the 4-row group
    rng = np.random.default_rng(seed)
    lengths = rng.choice([0, 1, 3, 17, 64, 65, 130, 300], size=n, p=[.1, .1, .2, .2, .15, .1, .1, .05])
    rows = np.repeat(np.arange(n), lengths)
    cols = rng.integers(0, n, rows.size)
    keep = cols != rows
    rows, cols = rows[keep], cols[keep]
    key = rows * n + cols
    _, first = np.unique(key, return_index=True)
    rows, cols = rows[first], cols[first]
    vals = 0.02 / np.sqrt(60.0) * rng.standard_normal(rows.size)
    d = np.cumsum(rng.uniform(0.8, 1.2, n))
    return ipt.Partition(d, ipt.CsrMatrix.from_triplets(n, n, rows, cols, vals))

def heavy(n, seed):
    # 1 % of the rows 200x longer than the rest: the upload cuts nonzero-balanced group ranges
    rng = np.random.default_rng(seed)
    lengths = np.where(rng.random(n) < 0.01, 2500, 12)
    rows = np.repeat(np.arange(n), lengths)
    cols = rng.integers(0, n, rows.size)
    keep = cols != rows
    rows, cols = rows[keep], cols[keep]
    key = rows * n + cols
    _, first = np.unique(key, return_index=True)
    rows, cols = rows[first], cols[first]
    vals = 0.3 / np.sqrt(2500.0) * rng.standard_normal(rows.size)
    d = np.cumsum(np.random.default_rng(seed + 1).uniform(0.8, 1.2, n))
    return ipt.Partition(d, ipt.CsrMatrix.from_triplets(n, n, rows, cols, vals))

out = {}
h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
cases = (("heavy16384", heavy(1 << 14, 3), 1e-12),) if sys.argv[2] == "heavy" else (
    ("ci4096", synth.csr_ci(4096, 32, 0.01, 42), 1e-10), ("ragged4099", ragged(4099, 5), 1e-12),
    ("ragged7", ragged(7, 2), 1e-12), ("ci65536", synth.csr_ci(65536, 32, 0.01, 7), 1e-10))
for name, p, tol in cases:
    g = ipt.build_gaps(p, 0.0)
    for anchor in (0, p.size() // 2):
        r = ipt.solve_single(p, g, anchor, ipt.IterationConfig(tolerance=tol, record_trace=True))
        out[f"{name}/{anchor}"] = [h(r.z), repr(r.eigenvalue), r.iterations, repr(r.final_step), repr(r.residual),
                                   h(np.asarray(r.trace)), int(r.status)]
    x = np.random.default_rng(1).standard_normal(p.size())
    out[f"{name}/matvec"] = h(ipt.kernels.matvec(p.delta, x))
    c = ipt.solve_single_continuation(p, g, 0, ipt.IterationConfig(tolerance=tol), 0.5)
    out[f"{name}/continuation"] = [h(c.z), repr(c.eigenvalue), c.iterations]
    acc = ipt.solve_single_accelerated(p, g, 0, ipt.IterationConfig(tolerance=tol), 3)
    out[f"{name}/accelerated"] = [h(acc.z), repr(acc.eigenvalue), acc.iterations]
print("RESULT " + json.dumps(out))
"""


def _run(variant, cases="plain"):
    env = dict(os.environ)
    env.pop("IPT_SPMV_VARIANT", None)
    if variant is not None:
        env["IPT_SPMV_VARIANT"] = str(variant)
    env.pop("IPT_SPMV_BALANCE", None)
    if cases == "plain":
        env["IPT_SPMV_BALANCE"] = "0"  # the ragged patterns stay on the round-robin kernels under test
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT, cases], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


@pytest.fixture(scope="module")
def default_run():
    return _run(None)


@pytest.mark.parametrize("variant", [16, 20, 24, 31])
def test_csr_map_kernels_agree_bit_for_bit(default_run, variant):
    other = _run(variant)
    assert other.keys() == default_run.keys()
    for k in default_run:
        assert other[k] == default_run[k], k


def test_balanced_ranges_agree_bit_for_bit():
    """Skewed rows: the default runs spmv_pipe_kernel over nonzero-balanced group ranges,
    variant 19 the group kernel over the same ranges."""
    a, b = _run(None, "heavy"), _run(19, "heavy")
    assert a.keys() == b.keys() and len(a) == 5
    for k in a:
        assert a[k] == b[k], k


def test_default_matches_numpy(default_run):
    # the default process also checks the plain matvec against numpy (1e-13 normwise)
    sys.path.insert(0, ROOT)
    import paper_2012_14702_b200 as ipt
    from paper_2012_14702_b200 import synth

    p = synth.csr_ci(4096, 32, 0.01, 42)
    x = np.random.default_rng(1).standard_normal(p.size())
    y = ipt.kernels.matvec(p.delta, x)
    rows = np.repeat(np.arange(p.size()), np.diff(p.delta.row_offsets))
    ref = np.zeros(p.size())
    np.add.at(ref, rows, p.delta.values * x[p.delta.col_indices])
    assert np.max(np.abs(y - ref)) <= 1e-13 * np.max(np.abs(ref))
    assert hashlib.sha256(np.ascontiguousarray(y).tobytes()).hexdigest() == default_run["ci4096/matvec"]


_CSCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import synth
h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
out = {}
for n in (4099, 65536):
    p = synth.csr_ci(n, 32, 0.01, 11)
    rp, ci, va = p.delta.row_offsets, p.delta.col_indices, p.delta.values
    rows = np.repeat(np.arange(n), np.diff(rp))
    vi = 0.003 * np.sign(ci - rows) * np.abs(va)  # antisymmetric imaginary part: Hermitian
    q = ipt.Partition(p.d, ipt.CsrMatrix(n, n, rp, ci, va + 1j * vi))
    r = ipt.solve_single(q, ipt.build_gaps(q, 0.0), 3, ipt.IterationConfig(tolerance=1e-11))
    out[f"hermitian{n}"] = [h(r.z), repr(r.eigenvalue), r.iterations, repr(r.residual)]
    x = np.random.default_rng(2).standard_normal(n) + 1j * np.random.default_rng(3).standard_normal(n)
    out[f"matvec{n}"] = h(ipt.kernels.matvec(q.delta, x))
    out[f"real_times_complex{n}"] = h(ipt.kernels.matvec(p.delta, x))
print("RESULT " + json.dumps(out))
"""


def _crun(kind):
    env = dict(os.environ)
    env.pop("IPT_CSPMV", None)
    if kind is not None:
        env["IPT_CSPMV"] = str(kind)
    r = subprocess.run([sys.executable, "-c", _CSCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


def test_complex_csr_kernels_agree_bit_for_bit():
    """cspmv_pipe_kernel (default, 3 entries per lane; 2) against cspmv_group_kernel."""
    base = _crun(None)
    assert len(base) == 6
    for kind in (0, 2):
        other = _crun(kind)
        for k in base:
            assert other[k] == base[k], (kind, k)
