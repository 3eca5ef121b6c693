"""Long randomised parity sweep against the reference build (tests/parity_fuzz.py):
    python tools/parity_sweep.py [first_seed] [count]
prints one line per failure and a per-entry-point summary (cases, worst eigenvector and
eigenvalue differences)."""
import collections
import os
import sys
import time
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import parity_fuzz  # noqa: E402
from parity_fuzz import draw, draw_cpp, draw_ext, run_case, run_case_cpp, run_case_ext  # noqa: E402

first = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
count = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
ext = len(sys.argv) > 3 and sys.argv[3] == "ext"
cpp = len(sys.argv) > 3 and sys.argv[3] == "cpp"
run, drawf = (run_case_ext, draw_ext) if ext else (run_case_cpp, draw_cpp) if cpp else (run_case, draw)
ref = oracle.ref()
stats = collections.defaultdict(lambda: [0, 0.0, 0.0, 0])
fails = 0
t0 = time.time()
for seed in range(first, first + count):
    try:
        kind, n, cplx, dz, dl = run(seed, ref)
        s = stats[(kind, cplx)]
        s[0] += 1
        s[1] = max(s[1], dz)
        s[2] = max(s[2], dl)
    except Exception as e:  # noqa: BLE001
        fails += 1
        dr = drawf(seed)
        kind, n, cplx, eps = dr[1], dr[2], dr[3], dr[-1]
        stats[(kind, cplx)][3] += 1
        print(f"FAIL seed {seed}: {kind} n={n} complex={cplx} eps={eps:.3g}: {type(e).__name__} {e}", flush=True)
        if os.environ.get("SWEEP_TRACE"):
            traceback.print_exc()
print(f"{count} cases (seeds {first}..{first + count - 1}), {fails} failures, {time.time() - t0:.0f} s")
print(f"{'entry point':16s} {'complex':7s} {'cases':>5s} {'fail':>4s} {'max |dZ|':>10s} {'max rel dLambda':>15s}")
for (kind, cplx), (c, dz, dl, f) in sorted(stats.items()):
    print(f"{kind:16s} {str(cplx):7s} {c:5d} {f:4d} {dz:10.2e} {dl:15.2e}")
if ext:
    c = parity_fuzz.STATUS_COUNTS
    print(f"reference statuses over the solves: converged {c[0]}, max_iterations {c[1]}, diverged {c[2]} "
          f"(the device matched each, iterations +-1)")
if os.environ.get("IPT_GUARD") == "1":
    import gc

    import paper_2012_14702_b200 as ipt

    gc.collect()
    lib = ipt.load_library()
    print(f"IPT_GUARD=1: guard zones checked on {lib.ipt_guard_checked()} buffers, "
          f"{lib.ipt_guard_violations()} violations")
