"""Key metrics per kernel launch of an ncu --set full report.
Usage: python tools/ncu_summary.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
W = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("launch__grid_size", "grid"),
     ("launch__block_size", "block"), ("launch__registers_per_thread", "regs"),
     ("smsp__inst_executed.sum", "warp_inst"), ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue%"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
     ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
     ("lts__t_bytes.sum", "l2_bytes"), ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
     ("l1tex__t_sector_hit_rate.pct", "l1hit%"), ("lts__t_sector_hit_rate.pct", "l2hit%"),
     ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
     ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wf%"),
     ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
     ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
     ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "lsb"),
     ("sm__cycles_elapsed.avg.per_second", "sm_hz")]
idx = [(h.index(k), n) for k, n in W if k in h]
units = rows[1]
for r in rows[2:]:
    out = []
    for i, n in idx:
        v = r[i]
        if n == "kernel":
            v = v.split("(")[0].replace("(anonymous namespace)::", "")[-40:]
        elif units[i] in ("Mbyte", "Gbyte", "Kbyte", "byte"):
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
            v = f"{float(v.replace(',', '')) * mult / 1e6:.1f}MB"
        elif units[i] == "nsecond":
            v = f"{float(v.replace(',', '')) / 1e3:.1f}"
        elif units[i] == "usecond":
            v = f"{float(v.replace(',', '')):.1f}"
        out.append(f"{n}={v}")
    print("  ".join(out))
