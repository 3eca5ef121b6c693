"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.md
    python tools/ncu_summary.py rep gpurun_out/prof_gemm_n8192.ncu-rep profiles/r01_ncu_gemm.md --flops 1.0995e12
    python tools/ncu_summary.py rep gpurun_out/prof_spmv.ncu-rep profiles/r01_ncu_spmv.md --bytes 1.66e9
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__occupancy_limit_registers",
]
UNIT_SCALE = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        sec = float(r[mi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1e-9)
        a = agg.setdefault(r[ki].split("(")[0][:80], [0, 0.0])
        a[0] += 1
        a[1] += sec
    tot = sum(v[1] for v in agg.values())
    lines = ["| launches | total ms | share | kernel |", "|---:|---:|---:|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {c} | {t * 1e3:.3f} | {100 * t / tot:.2f}% | `{k}` |")
    text = (f"ncu launch list ({os.path.basename(path)}): gpu__time_duration.sum per launch, "
            f"--clock-control none, cold-cache and serialised (compare shares, not absolutes).\n\n" + "\n".join(lines) + "\n")
    open(out, "w").write(text)
    print(text)


def rep(path, out, flops=None, nbytes=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for k in KEYS + ["Kernel Name"]:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (vals[i], units[i])
        res.append(d)
    lines = []
    summary = {}
    for d in res:
        name = d.get("Kernel Name", ("?", ""))[0]
        lines.append(f"### `{name[:120]}`\n")
        lines.append("| metric | value | unit |\n|---|---:|---|")
        for k in KEYS:
            if k in d:
                lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
        t = float(d["gpu__time_duration.sum"][0].replace(",", "")) * UNIT_SCALE.get(d["gpu__time_duration.sum"][1], 1e-9)
        rd = float(d["dram__bytes_read.sum"][0].replace(",", "")) * BYTES.get(d["dram__bytes_read.sum"][1], 1)
        wr = float(d["dram__bytes_write.sum"][0].replace(",", "")) * BYTES.get(d["dram__bytes_write.sum"][1], 1)
        summary = {"kernel": name, "time_s": t, "dram_bytes": rd + wr}
        if flops:
            lines.append(f"| achieved (algorithmic {flops:.4g} flop / time) | {flops / t / 1e12:.2f} | TFLOP/s |")
            summary["tflops"] = flops / t / 1e12
        if nbytes:
            lines.append(f"| achieved (algorithmic {nbytes:.4g} B / time) | {nbytes / t / 1e9:.0f} | GB/s |")
            lines.append(f"| dram traffic / algorithmic bytes | {(rd + wr) / nbytes:.3f} | x |")
            summary["gbs"] = nbytes / t / 1e9
        lines.append("")
    text = f"ncu --set full capture: {os.path.basename(path)}\n\n" + "\n".join(lines) + "\n"
    open(out, "w").write(text)
    print(text)
    return summary


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("kind", choices=["launches", "rep"])
    ap.add_argument("src")
    ap.add_argument("out")
    ap.add_argument("--flops", type=float)
    ap.add_argument("--bytes", type=float)
    a = ap.parse_args()
    if a.kind == "launches":
        launches(a.src, a.out)
    else:
        rep(a.src, a.out, a.flops, a.bytes)
