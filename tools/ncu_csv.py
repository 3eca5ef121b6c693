"""Print selected metrics of an ncu report (raw page) — helper for profiles/ summaries.

    python tools/ncu_csv.py gpurun_out/prof.ncu-rep [metric-substring ...]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
pats = sys.argv[2:] or ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
                        "launch__registers_per_thread", "launch__grid_size", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
                        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                        "l1tex__lsu_writeback_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
                        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                        "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank", "l1tex__t_output_wavefronts",
                        "l1tex__m_xbar2l1tex_read_sectors", "smsp__average_warp_latency_issue_stalled",
                        "smsp__pcsamp_warps_issue_stalled"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:110])
    for i, h in enumerate(hdr):
        if any(p in h for p in pats):
            print(f"  {h} = {r[i]} {units[i]}")
