"""Smoke-size workload for the memory-safety checks.

compute-sanitizer is closed on this GPU pool; the library's own guard zones stand in for
memcheck's out-of-bounds write detection (IPT_GUARD=1: 4 KB byte-pattern zones on both
sides of every device buffer, checked at release; tests/test_gpu_guard.py runs this script
that way and requires zero violations). Where compute-sanitizer is available:

    compute-sanitizer --tool memcheck  python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
    compute-sanitizer --tool synccheck python tools/sanitize_smoke.py

Covers every kernel family of the library at small sizes: the TMA/mbarrier DMMA GEMM
(full solve, map epilogue, closing product, identity-start map), the tcgen05 INT8 GEMM
and the Ozaki reconstruction (Ozaki solve), the matrix-free CG and the Cholesky fallback
of sigma_min, the dense LU with its cooperative panel kernel, the GEMV / grouped-CSR SpMV
maps with the fused step tail and the fused peer-store all-gather (stand-in peers), the
Anderson device path, the sparse-Delta SpMM map and the in-process communicator (2 ranks).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import _lib, dist, synth  # noqa: E402

lib = ipt.load_library()
cfg = ipt.IterationConfig(tolerance=1e-12)

p = synth.dense_uniform(300, 0.02, 42)
g = ipt.build_gaps(p)
r = ipt.solve_full(p, g, cfg)                                 # DMMA map + closing product + CG sigma_min
rz = ipt.solve_full(p, g, cfg, product="ozaki")               # tcgen05 INT8 GEMM + reconstruction
assert r.iterations == rz.iterations
os.environ["IPT_SIGMA"] = "factor"
ipt.smallest_singular_value_estimate(r.Z)                     # SYRK + blocked Cholesky path
del os.environ["IPT_SIGMA"]
w = np.eye(300) + 1e-3 * np.random.default_rng(1).standard_normal((300, 300))
ipt.solve_full(p, g, cfg, warm_start=w)                       # warm start (renormalise, GEMM map)

a = np.random.default_rng(2).standard_normal((200, 200)) + 1j * np.random.default_rng(3).standard_normal((200, 200))
f = ipt.lu_factor(a)                                          # cooperative LU panel kernel + DMMA updates
x = ipt.lu_solve(f, np.ones(200))

q = synth.csr_ci(4096, 16, 0.01, 7)
gq = ipt.build_gaps(q, 0.0)
s1 = ipt.solve_single(q, gq, 0, ipt.IterationConfig(tolerance=1e-10))    # grouped SpMV + fused tail
s2 = ipt.solve_single_accelerated(q, gq, 0, ipt.IterationConfig(residual_tolerance=1e-9), memory=3)
d4 = synth.dense_normal(1024)
s3 = ipt.solve_single(d4, ipt.build_gaps(d4), 0, cfg)                    # GEMV map + fused tail

# fused all-gather with stand-in peers (ipt_single_debug_peers)
import ctypes as C  # noqa: E402
from paper_2012_14702_b200._lib import Stats, check, dptr, i32ptr, i64ptr  # noqa: E402
from paper_2012_14702_b200.ipt import _params  # noqa: E402
ctx = ipt.default_context()
h = C.c_void_p()
check(lib.ipt_single_upload_csr(ctx.handle, 4096, dptr(q.d), None, i64ptr(q.delta.row_offsets),
                                i32ptr(q.delta.col_indices), dptr(q.delta.values), None, C.byref(h)))
check(lib.ipt_single_debug_peers(h, 3))
check(lib.ipt_single_reset(ctx.handle, h, 0, None, None))
st = Stats()
check(lib.ipt_single_iterate(ctx.handle, h, C.byref(_params(ipt.IterationConfig(tolerance=1e-10))), C.byref(st)))
lib.ipt_single_free(h)

sp = synth.csr_ci(1024, 8, 0.01, 3)
ipt.solve_full(sp, ipt.build_gaps(sp, 0.0), cfg)              # sparse-Delta SpMM map

ctxs = dist.local_contexts(2)                                 # in-process communicator, 2 ranks
outs = dist.run_ranks(lambda c: ipt.solve_full(p, g, cfg, ctx=c), ctxs)
assert np.array_equal(outs[0].Z, r.Z)
outs = dist.run_ranks(lambda c: ipt.solve_single(q, gq, 0, ipt.IterationConfig(tolerance=1e-10), ctx=c), ctxs)
assert np.array_equal(outs[0].z, s1.z)
for c in ctxs:
    c.close()
del outs, r, rz, s1, s2, s3, f
import gc  # noqa: E402

gc.collect()
ctx.close()
bad = lib.ipt_guard_violations()
print(f"sanitize smoke ok: {lib.ipt_kernel_launch_count()} kernel launches, guard zones checked on "
      f"{lib.ipt_guard_checked()} buffers, guard violations {bad}"
      f" (IPT_GUARD={os.environ.get('IPT_GUARD', '0')})")
sys.exit(1 if bad else 0)
