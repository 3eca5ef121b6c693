#!/usr/bin/env python3
"""Headline benchmark: full-spectrum IPT (BASELINE.json metric) on B200.

Workload (config.workload): BASELINE.json configs[2], full-spectrum IPT at
N = 32768, fp64, D = diag(1..N), Delta symmetric zero-diagonal uniform[-1,1]
(seed 42), eps = 0.32/sqrt(N), Z column-sharded over the ranks with Delta
replicated (strong scaling: the same N for every GPU count). Synthetic data of
exactly that construction (there is no dataset in the reference).

A "step" is one IPT iteration (one map application F(Z)): K2 diagonal
pre-pass + K1 fused DMMA GEMM/map epilogue + fixed-order reduction (+ NCCL
all-reduce of the step scalars for N>1) + device-side stop decision. `value` is
whole-job FP64 TFLOP/s = 2 N^3 per step / step time (max over ranks), inputs
resident in HBM. `e2e` is the same metric through the drop-in C ABI
(ipt_full_solve) with host buffers: H2D of Delta, the iterations to
convergence, the closing product, sigma_min, and D2H of Z and Lambda.

Secondary lines (same JSON object, "secondary"): the single-eigenpair paths
(config 4 dense GEMV at N = 65536 and config 5 CSR SpMV at N = 2^21) in GB/s.

`--impl reference` times the reference's own CPU implementation (oracle/_ref,
built from the reference sources) on the host cores instead.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_FULL = 32768
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
DMMA_ISSUE_PEAK = 37.1  # TF/s, FP64 DMMA issue-rate microbenchmark on this pool (profiles/r01_fp64_probe.txt)
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")
METRIC = "IPT full-spectrum FP64 TFLOP/s (2N^3 per iteration), N=32768"


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def workload_config(world, n, extra=None):
    cfg = {
        "workload": f"BASELINE configs[2]: full-spectrum IPT fp64 dense symmetric N={n}, D=diag(1..N), "
                    f"Delta uniform[-1,1] symmetric zero-diagonal, eps=0.32/sqrt(N), Z column-sharded over "
                    f"{world} GPU(s), Delta replicated",
        "n": n,
        "eps": 0.32 / math.sqrt(n),
        "seed": 42,
        "step": "one IPT map application (diag pre-pass + fused DMMA GEMM/epilogue + reduction + stop decision)",
        "parallelism": f"column-shard x{world}" if world > 1 else "single GPU",
        "l2": "inputs exceed L2 (Delta 8.6 GB, Z 8.6 GB per buffer vs 126 MB L2); no flush needed",
    }
    if extra:
        cfg.update(extra)
    return cfg


# --------------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi equivalent via NVML: SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self.stop_ev.wait(0.2)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- peaks


def fp64_peak(torch):
    """cuBLAS DGEMM (torch float64 matmul) 8192^3 best of 5: the FP64 denominator.
    MEASURED_PEAKS.json carries no FP64 figure; this is measured on the same GPU in
    the same run (burst), beside the DMMA issue-rate probe (profiles/r01_fp64_probe.txt)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / best / 1e12


def hbm_peak():
    try:
        return json.load(open(PEAKS_PATH))["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_for(kernel, n=None):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed
    ncu --set full capture (profiles/ncu_traffic.json), when it was taken at this size."""
    try:
        rec = json.load(open(TRAFFIC_PATH)).get(kernel)
    except Exception:
        return None
    if rec is None or (n is not None and rec.get("n") != n):
        return None
    return rec.get("dram_bytes_per_launch")


# --------------------------------------------------------------------------- CPU baseline


def use_all_host_threads():
    """The reference's OpenMP on every host core (torchrun exports OMP_NUM_THREADS=1 to
    each rank; torch may have initialised libgomp already): the environment for libraries
    loaded later, and the calling thread's ICV for the one already loaded."""
    threads = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(threads)
    try:
        C.CDLL("libgomp.so.1").omp_set_num_threads(threads)
    except OSError:
        pass
    return threads


def cpu_reference_sample(n=4096, reps=2):
    """The reference's own apply_map_full (solver.cpp:156-178; kernels.cpp dgemm) on the
    host cores, one map application at a bounded N of the same construction."""
    import oracle

    use_all_host_threads()
    d, delta = oracle.port().dense_uniform(n, 0.32 / math.sqrt(n), 42)  # no product library here
    if oracle.have_ref():
        R, kind = oracle.ref(), "reference"

        def step(z):
            return R.apply_map_full(d, delta, z)
    else:  # reference build absent: the plain-C restatement of the same map
        P, kind = oracle.port(), "port"

        def step(z):
            return P.full_map_block(d, delta, 0, z)[0]
    z = step(np.eye(n))  # warm
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        z = step(z)
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    return {"value": 2.0 * n ** 3 / t / 1e12, "unit": "TFLOP/s", "cores": int(os.environ["OMP_NUM_THREADS"]),
            "kind": kind,
            "sample": f"{kind} apply_map_full (one IPT iteration) at N={n}, same construction, "
                      f"best of {reps}: {t:.3f} s; metric counts 2N^3 useful flops"}


def per_config_e2e(ipt, ctx):
    """End-to-end time to solution of the configs the reference runs whole on the host
    (BASELINE configs[0]: full spectrum N=1024; configs[4]: CSR single pair N=2^21): the
    drop-in call with host buffers on the B200 vs the reference build's own solve on all
    host cores, same inputs and stop rule (configs 1, 2, 5 run end to end;
    config 2 needs ~15 min per reference iteration here, so it is left out)."""
    import oracle
    from paper_2012_14702_b200 import synth

    if not oracle.have_ref():
        return {"error": "reference build absent (oracle/_ref)"}
    R = oracle.ref()
    out = {"cores": use_all_host_threads()}
    p1 = synth.config1()
    cfg1 = ipt.IterationConfig(tolerance=1e-12)
    ipt.solve_full(p1, ipt.build_gaps(p1), cfg1, ctx=ctx)  # warm
    t0 = time.perf_counter()
    g1 = ipt.solve_full(p1, ipt.build_gaps(p1), cfg1, ctx=ctx)
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    r1 = R.solve_full(p1.d, p1.delta, tol=1e-12)
    tr = time.perf_counter() - t0
    out["config1_full_n1024"] = {
        "gpu_s": tg, "reference_s": tr, "reference_inner_s": r1["seconds"], "speedup": r1["seconds"] / tg,
        "iterations": [g1.iterations, r1["iterations"]],
        "lambda0_rel_diff": abs(float(g1.eigenvalues[0]) - r1["eigenvalues"][0].real) / abs(r1["eigenvalues"][0].real)}
    del p1, g1, r1
    p5 = synth.config5()
    g5gaps = ipt.build_gaps(p5, 0.0)
    cfg5 = ipt.IterationConfig(tolerance=1e-10)
    ipt.solve_single(p5, g5gaps, 0, cfg5, ctx=ctx)  # warm (pools, staging), as for config 1
    tg_all = []
    for _ in range(3):  # host-side staging of 1.6 GB varies run to run (58-130 ms): median of three calls
        t0 = time.perf_counter()
        g5 = ipt.solve_single(p5, g5gaps, 0, cfg5, ctx=ctx)
        tg_all.append(time.perf_counter() - t0)
    tg = sorted(tg_all)[1]
    t0 = time.perf_counter()
    r5 = R.solve_single(p5.d, p5.delta, 0, tol=1e-10, degeneracy_tol=0.0)
    tr = time.perf_counter() - t0
    out["config5_csr_single_n2097152"] = {
        "gpu_s": tg, "gpu_s_all": tg_all, "reference_s": tr, "reference_inner_s": r5["seconds"],
        "speedup": r5["seconds"] / tg, "iterations": [g5.iterations, r5["iterations"]],
        "eigenvalue_rel_diff": abs(g5.eigenvalue - r5["eigenvalue"].real) / abs(r5["eigenvalue"].real),
        "note": "gpu_s: the drop-in call with host buffers (H2D of the 1.6 GB CSR arrays included); "
                "reference_inner_s: the reference solve itself (its timer, inputs already in its CSR "
                "ComplexMatrix); speedup = reference_inner_s / gpu_s"}
    return out


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import oracle

    n = args.ref_n
    use_all_host_threads()  # every host core, also under torchrun (OMP_NUM_THREADS=1 there)
    # Inputs from the reference's generator restated in the oracle (rng.hpp, SURVEY 8(d)
    # draw order): this process loads only oracle/ libraries, never libipt_b200.so.
    d, delta = oracle.port().dense_uniform(n, 0.32 / math.sqrt(n), 42)
    if oracle.have_ref():  # the reference's own apply_map_full (oracle/_ref, built from its sources)
        R = oracle.ref()
        kind = "reference"

        def step(z):
            return R.apply_map_full(d, delta, z)
    else:  # the plain-C restatement of the same map (oracle/ipt_oracle.c)
        P = oracle.port()
        kind = "port"

        def step(z):
            return P.full_map_block(d, delta, 0, z)[0]
    z = np.eye(n, dtype=np.complex128)
    for _ in range(args.warmup):
        z = step(z)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        z = step(z)
    t = time.perf_counter() - t0
    value = 2.0 * n ** 3 * args.steps / t / 1e12
    ref_config = workload_config(world, N_FULL, {"reference_sample_n": n, "same_config": False})
    ref_config["workload"] += (f" | reference arm: each step is ONE reference apply_map_full at the bounded "
                               f"sample N={n} of the same construction (reference_sample_n), rate per 2N^3 flops")
    sample = (f"reference apply_map_full (proj/src/solver.cpp:156-178, OpenMP kernels.cpp) at N={n} of the "
              f"same construction per step (the N={N_FULL} workload needs ~120 GB and hours per iteration "
              f"on the CPU); metric counts 2N^3 flops per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": max(world, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": ref_config,
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": int(os.environ["OMP_NUM_THREADS"]),
                         "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- secondary: single pair


def bench_single(ipt, lib, ctx, which, steps, warmup, hbm, reduce_max=lambda x: x, world=1):
    from paper_2012_14702_b200 import synth
    from paper_2012_14702_b200._lib import check, dptr, i32ptr, i64ptr

    t0 = time.perf_counter()
    if which == "gemv":
        n = 65536
        p = synth.config4()
        nbytes = 8.0 * n * n + 3 * 8.0 * n
        h = C.c_void_p()
        check(lib.ipt_single_upload_dense(ctx.handle, n, dptr(p.d), None, dptr(p.delta), None, C.byref(h)))
        kernel = "gemv_map_kernel<1>"
        tol = 1e-12
        gaps_tol = -1.0
    else:
        n = 1 << 21
        p = synth.config5()
        nnz = p.delta.nnz
        nbytes = 12.0 * nnz + 8.0 * (n + 1) + 3 * 8.0 * n
        h = C.c_void_p()
        check(lib.ipt_single_upload_csr(ctx.handle, n, dptr(p.d), None, i64ptr(p.delta.row_offsets),
                                        i32ptr(p.delta.col_indices), dptr(p.delta.values), None, C.byref(h)))
        kernel = "spmv_pipe_kernel<1, 3, 4, 1>"
        tol = 1e-10
        gaps_tol = 0.0
    setup_s = time.perf_counter() - t0
    # a real solve for the time-to-convergence line
    check(lib.ipt_single_reset(ctx.handle, h, 0, None, None))
    from paper_2012_14702_b200._lib import Stats
    from paper_2012_14702_b200.ipt import _params

    prm = _params(ipt.IterationConfig(tolerance=tol))
    st = Stats()
    check(lib.ipt_single_iterate(ctx.handle, h, C.byref(prm), C.byref(st)))
    check(lib.ipt_single_finalize(ctx.handle, h, C.byref(st)))
    solve = {"iterations": st.iterations, "status": ipt.to_string(st.status), "eigenvalue": st.eigenvalue_re,
             "residual": st.residual, "loop_ms": st.ms_loop, "final_ms": st.ms_final}
    check(lib.ipt_single_reset(ctx.handle, h, 0, None, None))
    tot, dom = C.c_double(), C.c_double()
    check(lib.ipt_single_run_steps(ctx.handle, h, warmup, C.byref(tot), C.byref(dom)))
    check(lib.ipt_single_run_steps(ctx.handle, h, steps, C.byref(tot), C.byref(dom)))
    lib.ipt_single_free(h)
    step_ms = reduce_max(tot.value / steps)
    dom_ms_local = dom.value / steps
    dom_ms = reduce_max(dom_ms_local)
    solve["loop_ms"] = reduce_max(solve["loop_ms"])
    kbytes = nbytes - 8.0 * n  # the map kernel itself: matrix + z + d + fz
    del p
    out = {
        "workload": ("configs[3] dense GEMV single pair N=65536" if which == "gemv"
                     else f"configs[4] CSR SpMV single pair N=2^21 (~64 nnz/row), rows sharded over {world} "
                          f"GPU(s) (strong scaling), fused peer-store all-gather of the iterate"),
        "n_gpus": world,
        "metric": "single-pair IPT iteration GB/s (algorithmic bytes)",
        "value": nbytes / (step_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": step_ms,
        "time_to_solution": solve, "setup_s": setup_s,
        "roofline": {"bound": "hbm", "kernel": kernel, "achieved": kbytes / (dom_ms * 1e-3) / 1e9,
                     "peak": hbm[0], "peak_source": hbm[1], "unit": "GB/s",
                     "frac": kbytes / (dom_ms * 1e-3) / 1e9 / hbm[0], "kernel_ms": dom_ms,
                     "bytes_per_launch": kbytes, "traffic": traffic_for(kernel, n)},
    }
    if world > 1:  # per-rank kernel bytes: this rank's rows (a 1/world share of the matrix stream)
        out["roofline"]["achieved"] = kbytes / world / (dom_ms_local * 1e-3) / 1e9
        out["roofline"]["frac"] = out["roofline"]["achieved"] / hbm[0]
        out["roofline"]["bytes_per_launch"] = kbytes / world
    if which == "spmv":
        # The random z gather (32-byte L2 sector per 8-byte use), not HBM, bounds this
        # kernel: measured ceiling = the same stream + gather without row structure.
        ceil_ms = 0.518
        out["roofline"]["memory_ceiling"] = {
            "ms": ceil_ms, "frac": ceil_ms / dom_ms,
            "source": "profiles/r01_gather_probe.txt (tools/probes/gather_probe.cu, one B200)"}
    return out


def cpp_dropin_phases():
    """The C++ drop-in API (include/ipt/*.hpp) timed with the reference's own phase method
    (proj/src/bench.cpp:50-99, medians of the repetitions) by tools/cpp/dropin_bench: the
    caller's std::complex ComplexMatrix carriers in and out, so the layout conversion at
    the boundary is inside every number."""
    import subprocess

    exe = os.path.join(ROOT, "tools", "cpp", "dropin_bench")
    if not os.path.exists(exe):
        return {"error": "tools/cpp/dropin_bench not built (make -C paper_2012_14702_b200)"}
    out = {"method": "proj/src/bench.cpp:50-99 phases through ipt::solve_full / solve_single / kernels:: (C++)"}
    for cfg, reps in (("2", "3"), ("5", "3"), ("3", "2")):
        try:
            r = subprocess.run([exe, cfg, reps], capture_output=True, text=True, timeout=900)
            line = [x for x in r.stdout.splitlines() if x.startswith("{")]
            out[f"config{cfg}"] = json.loads(line[-1]) if line else {"error": r.stderr[-300:]}
        except Exception as exc:  # report, never hide
            out[f"config{cfg}"] = {"error": repr(exc)}
    return out


def bench_sparse_full(lib, ctx, n, per_row, steps, dense_step_ms):
    """Sparse-Delta full map: CSR Delta with per_row entries per row at the
    headline N, fused SpMM map (spmm_full_kernel<0,4>), Z row-major in HBM. Bound: the
    L2->SM gather of nnz * N * 8 bytes per map (the Z chunk in flight stays in L2)."""
    from paper_2012_14702_b200._lib import check, dptr, i32ptr, i64ptr

    rng = np.random.default_rng(7)
    cols = np.sort(rng.integers(0, n, (n, per_row)), axis=1).astype(np.int32)
    vals = 0.01 * rng.standard_normal((n, per_row))
    vals[cols == np.arange(n)[:, None]] = 0.0
    rowptr = np.arange(0, n * per_row + 1, per_row, dtype=np.int64)
    d = np.arange(n, dtype=float)
    h = C.c_void_p()
    check(lib.ipt_full_upload_csr(ctx.handle, n, dptr(d), None, i64ptr(rowptr), i32ptr(cols.ravel()),
                                  dptr(vals.ravel()), None, C.byref(h)))
    check(lib.ipt_full_reset(ctx.handle, h, None, None))
    tot, ker = C.c_double(), C.c_double()
    check(lib.ipt_full_run_maps(ctx.handle, h, 3, C.byref(tot), C.byref(ker)))
    check(lib.ipt_full_run_maps(ctx.handle, h, steps, C.byref(tot), C.byref(ker)))
    lib.ipt_full_free(h)
    nnz = n * per_row
    ms = tot.value / steps
    ms_k = ker.value / steps
    gather = nnz * n * 8.0
    return {"workload": f"sparse Delta full map N={n}, {per_row} nnz/row (random columns), Z row-major",
            "ms_per_map": ms, "kernel_ms": ms_k, "kernel": "spmm_full_kernel<0,4>",
            "gather_bytes_per_launch": gather, "gather_TBps": gather / (ms_k * 1e-3) / 1e12,
            "roofline_note": "L2 (LTS) bound: ~6300 B/clk full chip (B300_MICROARCH.md) ~ 12 TB/s",
            "speedup_vs_dense_map": dense_step_ms / ms if dense_step_ms else None}


def int8_peak():
    """Dense INT8 tensor peak for the roofline: twice MEASURED_PEAKS' bf16 figures (the
    tcgen05 kind::i8 rate is 2x kind::f16 per SM per clock), burst and sustained."""
    try:
        pk = json.load(open(PEAKS_PATH))
        return 2.0 * pk["bf16_tflops"], 2.0 * pk.get("bf16_tflops_sustained", pk["bf16_tflops"]), \
            "2 x MEASURED_PEAKS.json bf16_tflops (burst) / bf16_tflops_sustained"
    except Exception:
        return 4500.0, 4500.0, "nominal dense INT8 4.5 POPS (B200_PROFILING.md fallback)"


def bench_ozaki(ipt, lib, ctx, n, dense_step_ms, dmma_solve):
    """The same map and solve with W = Delta Z by Ozaki scheme II on the tcgen05 INT8
    datapath (16 exact modular GEMMs + CRT reconstruction, ozaki.cu): FP64-accurate, so
    reported with its agreement to the DMMA (FP64 tensor core) solve. The roofline kernel
    is the INT8 GEMM (i8gemm_2sm_kernel), timed with events around its 16 launches per map."""
    from paper_2012_14702_b200 import synth
    from paper_2012_14702_b200._lib import check, dptr

    p = synth.config3(n=n)
    h = C.c_void_p()
    check(lib.ipt_full_upload(ctx.handle, n, dptr(p.d), None, dptr(p.delta), None, C.byref(h)))
    check(lib.ipt_full_reset(ctx.handle, h, None, None))
    check(lib.ipt_full_set_product(h, 1))
    tot, ker = C.c_double(), C.c_double()
    check(lib.ipt_full_run_maps(ctx.handle, h, 2, C.byref(tot), C.byref(ker)))
    steps = 3
    check(lib.ipt_full_run_maps(ctx.handle, h, steps, C.byref(tot), C.byref(ker)))
    moduli = C.c_int32()
    check(lib.ipt_full_ozaki_moduli(h, C.byref(moduli)))
    lib.ipt_full_free(h)
    ms = tot.value / steps
    gemm_ms = ker.value / steps
    int8_ops = moduli.value * 2.0 * n ** 3  # one 2N^3 int8 GEMM per modulus in use (Z_jj split off)
    burst, sustained, src = int8_peak()
    achieved = int8_ops / (gemm_ms * 1e-3) / 1e12
    t0 = time.perf_counter()
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12), ctx=ctx, product="ozaki")
    tts = time.perf_counter() - t0
    out = {"workload": f"configs[2] N={n}, W = Delta Z by Ozaki scheme II on tcgen05 kind::i8 "
                       f"({moduli.value} of 16 moduli after splitting off Z_jj)",
           "moduli": moduli.value,
           "ms_per_map": ms, "fp64_equivalent_TFs": 2.0 * n ** 3 / (ms * 1e-3) / 1e12,
           "speedup_vs_dmma_map": dense_step_ms / ms,
           "roofline": {"bound": "tensor", "kernel": f"i8gemm_2sm_kernel<ModStore, 2> ({moduli.value} launches per map)",
                        "achieved": achieved, "peak": burst, "peak_sustained": sustained, "unit": "TOPS (int8)",
                        "frac": achieved / burst, "frac_of_sustained": achieved / sustained,
                        "ops_per_map": int8_ops, "gemm_ms_per_map": gemm_ms,
                        "gemm_share_of_map": gemm_ms / ms, "peak_source": src},
           "time_to_solution_s": tts, "iterations": r.iterations, "status": ipt.to_string(r.status),
           "timings_ms": r.timings_ms, "residual_frobenius": r.residual_frobenius}
    if dmma_solve is not None and dmma_solve.get("lambda0") is not None:
        out["lambda0"] = float(r.eigenvalues[0])
        out["lambda0_rel_diff_vs_dmma"] = abs(float(r.eigenvalues[0]) - dmma_solve["lambda0"]) / abs(dmma_solve["lambda0"])
    return out


def shared_outputs(n, rank, barrier):
    """Full-size Z / eigenvalue host arrays mapped by every rank (/dev/shm), for the
    column-local output of a sharded solve; None when /dev/shm cannot hold them."""
    import shutil

    need = 8 * n * n + 8 * n
    tag = os.environ.get("MASTER_PORT", "0")
    paths = [f"/dev/shm/ipt_bench_{tag}_z", f"/dev/shm/ipt_bench_{tag}_lam"]
    ok = [0]
    if rank == 0:
        try:
            ok[0] = int(shutil.disk_usage("/dev/shm").free > 1.2 * need)
        except OSError:
            ok[0] = 0
        if ok[0]:
            np.memmap(paths[0], dtype=np.float64, mode="w+", shape=(n, n)).flush()
            np.memmap(paths[1], dtype=np.float64, mode="w+", shape=(n,)).flush()
    import torch
    import torch.distributed as dist

    t = torch.tensor(ok, dtype=torch.int32, device="cuda")
    dist.broadcast(t, 0)
    barrier()
    if not int(t.item()):
        return None, None
    zr = np.memmap(paths[0], dtype=np.float64, mode="r+", shape=(n, n))
    lr = np.memmap(paths[1], dtype=np.float64, mode="r+", shape=(n,))
    return (zr, None, lr, None), paths


# --------------------------------------------------------------------------- launch


def relaunch_if_needed(args):
    """`--gpus N` (N > 1) outside torchrun: re-launch this command as N ranks under
    torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous); fail loudly when
    fewer than N GPUs are visible. Returns an exit code, or None to run in-process."""
    world = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if world:
        if args.gpus > 1 and world != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
            return 2
        return None
    if args.gpus <= 1 or args.impl == "reference":
        return None  # the reference arm is CPU work on rank 0 only
    import socket
    import subprocess

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible",
              file=sys.stderr)
        return 3
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# --------------------------------------------------------------------------- main arm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=N_FULL)
    ap.add_argument("--ref-n", type=int, default=4096)
    ap.add_argument("--secondary", default="all", choices=["all", "none", "gemv", "spmv"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    rc = relaunch_if_needed(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2012_14702_b200 as ipt
    from paper_2012_14702_b200 import dist as idist
    from paper_2012_14702_b200 import synth
    from paper_2012_14702_b200._lib import check, dptr

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = idist.init_context_from_env()
    lib = ipt.load_library()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    peak = fp64_peak(torch) if rank == 0 else 0.0
    # FP64 DMMA issue rate measured in this run by the library's probe (m16n8k4 from
    # registers on every SM); the round-1 pool constant is only a fallback
    dmma_probe = None
    if rank == 0:
        v = C.c_double()
        if lib.ipt_fp64_issue_probe(ctx.handle, C.byref(v)) == 0:
            dmma_probe = v.value
    fp64_den = max(peak, dmma_probe if dmma_probe else DMMA_ISSUE_PEAK)
    n = args.n
    t0 = time.perf_counter()
    p = synth.config3(n=n)
    gen_s = time.perf_counter() - t0

    # ---------------- device-resident timed steps
    h = C.c_void_p()
    check(lib.ipt_full_upload(ctx.handle, n, dptr(p.d), None, dptr(p.delta), None, C.byref(h)))
    check(lib.ipt_full_reset(ctx.handle, h, None, None))
    c0, c1 = C.c_int64(), C.c_int64()
    lib.ipt_full_local_columns(h, C.byref(c0), C.byref(c1))
    ncols = c1.value - c0.value
    tot, gem = C.c_double(), C.c_double()
    check(lib.ipt_full_run_maps(ctx.handle, h, args.warmup, C.byref(tot), C.byref(gem)))
    launches0 = lib.ipt_kernel_launch_count()
    barrier()
    wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        check(lib.ipt_full_run_maps(ctx.handle, h, args.steps, C.byref(tot), C.byref(gem)))
    barrier()
    wall = time.perf_counter() - wall0
    launches = lib.ipt_kernel_launch_count() - launches0
    step_ms = max_over_ranks(tot.value / args.steps)
    gemm_ms_local = gem.value / args.steps
    gemm_ms = max_over_ranks(gemm_ms_local)
    lib.ipt_full_free(h)
    flops_step = 2.0 * n ** 3
    value = flops_step / (step_ms * 1e-3) / 1e12
    gemm_flops_local = 2.0 * n * n * ncols
    achieved = gemm_flops_local / (gemm_ms_local * 1e-3) / 1e12

    # ---------------- end to end through the C ABI with host buffers
    e2e = None
    solve_info = None
    if not args.no_e2e:
        torch.cuda.empty_cache()
        barrier()
        # N > 1: every rank writes its own columns of Z into one shared host array
        # (IPT_OUTPUT_LOCAL_COLUMNS, a /dev/shm mapping), no gather through rank 0
        out, shm = None, None
        if world > 1:
            out, shm = shared_outputs(n, rank, barrier)
        # one untimed solve first (device pools, pinned staging and the host result pages
        # of this process warm), like the W warm-up steps of `value`
        ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12), ctx=ctx,
                       output="local" if out is not None else "root", out=out)
        barrier()
        t0 = time.perf_counter()
        gaps = ipt.build_gaps(p)
        t_gaps = time.perf_counter() - t0
        r = ipt.solve_full(p, gaps, ipt.IterationConfig(tolerance=1e-12), ctx=ctx,
                           output="local" if out is not None else "root", out=out)
        t_call = time.perf_counter() - t0 - t_gaps
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        if os.environ.get("IPT_PROFILE"):
            print(f"[bench] e2e: build_gaps {1e3 * t_gaps:.1f} ms, solve_full {1e3 * t_call:.1f} ms, "
                  f"total {1e3 * e2e_s:.1f} ms", file=sys.stderr, flush=True)
        e2e = {"value": flops_step * r.iterations / e2e_s / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(8 * n * n + 8 * n),
               "d2h_bytes_per_step": int(8 * n * n + 8 * n),
               "step": "one drop-in solve_full call (C ABI ipt_full_solve, host buffers, pageable memory); "
                       "h2d / d2h bytes are the whole job's (with g GPUs each rank uploads 1/g of Delta's rows "
                       "and an NVLink all-gather replicates it; each rank downloads its own columns of Z into "
                       "a shared host mapping when output is local)",
               "output": "local columns (shared /dev/shm mapping)" if out is not None else "root",
               "seconds": e2e_s,
               "warmup_calls": 1,
               "flop_convention": "2N^3 per IPT iteration (the metric's definition) x iterations / wall time: a "
                                  "work rate in the reference's units, not an executed-FLOP rate (it can exceed the "
                                  "FP64 peak). Executed: iterations-1 FP64 map GEMMs (the first map from Z = I needs "
                                  "no product: W = Delta I = Delta bit for bit) and, for the closing residual, the "
                                  "last map's product plus an INT8 tensor-core correction Delta (Z_new - Z_old) "
                                  "(K16: two INT8 GEMMs, K and 2K long) instead of one more FP64 GEMM; the "
                                  "reference executes iterations+1 FP64-complex products",
               "gemms_executed": {"fp64_map": int(r.iterations) - 1,
                                  "int8_closing_correction": 2 if r.timings_ms.get("final", 1e9) < 0.2 * r.timings_ms.get("loop", 0) / max(1, int(r.iterations) - 1) else 0,
                                  "fp64_closing": 0 if r.timings_ms.get("final", 1e9) < 0.2 * r.timings_ms.get("loop", 0) / max(1, int(r.iterations) - 1) else 1}}
        solve_info = {"iterations": r.iterations, "status": ipt.to_string(r.status),
                      "residual_frobenius": r.residual_frobenius,
                      "residual_rel": r.residual_frobenius / math.sqrt(float(np.sum(p.delta ** 2)) + float(np.sum(p.d ** 2))),
                      "sigma_min": r.min_singular_value_estimate, "timings_ms": r.timings_ms,
                      "time_to_solution_s": e2e_s,
                      "lambda0": float(r.eigenvalues[0]) if rank == 0 else None}
        del r
        if shm is not None:
            barrier()
            del out
            if rank == 0:
                for f in shm:
                    try:
                        os.unlink(f)
                    except OSError:
                        pass
    del p

    # ---------------- secondary: single-pair paths (rank 0, N = 1 only)
    secondary = {}
    if args.secondary != "none":
        hbm = hbm_peak()
        # config 4 (dense GEMV) is "replicas only"; config 5 (CSR) is row-sharded
        kinds = ["gemv", "spmv"] if args.secondary == "all" else [args.secondary]
        for which in [k for k in kinds if world == 1 or k == "spmv"]:
            try:
                barrier()
                secondary[which] = bench_single(ipt, lib, ctx, which, max(args.steps, 10), 3, hbm,
                                                max_over_ranks, world)
            except Exception as exc:  # report, never hide
                secondary[which] = {"error": repr(exc)}
    if world == 1 and args.secondary != "none":
        if args.secondary == "all":
            try:  # the low end of the metric's N range: configs[1], N = 8192, through the C ABI
                p2 = synth.config2()
                ipt.solve_full(p2, ipt.build_gaps(p2), ipt.IterationConfig(tolerance=1e-12), ctx=ctx)  # warm
                t0 = time.perf_counter()
                r2 = ipt.solve_full(p2, ipt.build_gaps(p2), ipt.IterationConfig(tolerance=1e-12), ctx=ctx)
                t2 = time.perf_counter() - t0
                secondary["full_n8192"] = {
                    "workload": "configs[1] full spectrum N=8192, eps=0.32/sqrt(N), tol 1e-12 (C ABI, host buffers)",
                    "time_to_solution_s": t2, "iterations": r2.iterations, "status": ipt.to_string(r2.status),
                    "e2e_tflops": 2.0 * 8192 ** 3 * r2.iterations / t2 / 1e12,
                    # executed map GEMMs: the first map from Z = I needs no product (W = Delta I)
                    "loop_gemms_executed": r2.iterations - 1,
                    "loop_tflops": 2.0 * 8192 ** 3 * (r2.iterations - 1) / (r2.timings_ms["loop"] * 1e-3) / 1e12,
                    "timings_ms": r2.timings_ms, "lambda0": float(r2.eigenvalues[0]),
                    "residual_frobenius": r2.residual_frobenius, "sigma_min": r2.min_singular_value_estimate}
                # the same solve with the Ozaki product (tcgen05 INT8)
                ipt.solve_full(p2, ipt.build_gaps(p2), ipt.IterationConfig(tolerance=1e-12), ctx=ctx,
                               product="ozaki")  # warm
                t0 = time.perf_counter()
                r3 = ipt.solve_full(p2, ipt.build_gaps(p2), ipt.IterationConfig(tolerance=1e-12), ctx=ctx,
                                    product="ozaki")
                t3 = time.perf_counter() - t0
                secondary["full_n8192"]["ozaki"] = {
                    "time_to_solution_s": t3, "iterations": r3.iterations, "status": ipt.to_string(r3.status),
                    "e2e_tflops_fp64_equivalent": 2.0 * 8192 ** 3 * r3.iterations / t3 / 1e12,
                    "timings_ms": r3.timings_ms, "lambda0": float(r3.eigenvalues[0]),
                    "residual_frobenius": r3.residual_frobenius}
                del p2, r2, r3
            except Exception as exc:
                secondary["full_n8192"] = {"error": repr(exc)}
            try:
                secondary["sparse_full"] = bench_sparse_full(lib, ctx, n, 64, max(args.steps, 5), step_ms)
            except Exception as exc:
                secondary["sparse_full"] = {"error": repr(exc)}
            try:
                secondary["ozaki"] = bench_ozaki(ipt, lib, ctx, n, step_ms, solve_info)
            except Exception as exc:
                secondary["ozaki"] = {"error": repr(exc)}

    if world == 1 and args.secondary == "all":
        lib.ipt_ctx_trim(ctx.handle)  # the subprocess needs the device memory this process keeps cached
        torch.cuda.empty_cache()
        secondary["cpp_dropin"] = cpp_dropin_phases()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference_sample()
        except Exception as exc:
            cpu = {"error": repr(exc)}
        if args.secondary == "all":
            try:
                secondary["per_config_e2e_vs_reference"] = per_config_e2e(ipt, ctx)
            except Exception as exc:
                secondary["per_config_e2e_vs_reference"] = {"error": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE configs[2] construction, seed 42)",
            "config": workload_config(world, n),
            "roofline": {"bound": "tensor", "kernel": "dmma_tma_kernel<1> (K1: TMA-fed DMMA GEMM + fused map epilogue)",
                         "achieved": achieved, "peak": fp64_den,
                         "peak_source": "FP64 tensor peak (absent from MEASURED_PEAKS.json): the larger of the DMMA "
                                        "issue-rate probe (ipt_fp64_issue_probe: m16n8k4 DMMAs from registers on "
                                        "every SM) and cuBLAS DGEMM 8192^3, both measured in this run"
                                        + ("" if dmma_probe else " (probe failed: pool constant 37.1 TF/s, "
                                           "profiles/r01_fp64_probe.txt)"),
                         "dmma_issue_probe_in_run": dmma_probe,
                         "cublas_dgemm_in_run": peak,
                         "unit": "TFLOP/s", "frac": achieved / fp64_den,
                         "frac_of_cublas_dgemm": achieved / peak if peak else None,
                         "flops_per_launch": gemm_flops_local, "kernel_ms": gemm_ms_local,
                         "kernel_share_of_step": gemm_ms / step_ms,
                         "traffic": traffic_for("dmma_tma_kernel<1>", n) if world == 1 else None},
            "time_to_solution": solve_info,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "wall_s_timed": wall,
            "setup": {"generate_s": gen_s},
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
