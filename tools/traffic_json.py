"""profiles/traffic_<WL>.json from an `ncu --set full` report of one bench step: DRAM bytes
(read + write) per launch of K1c (k1_packed / k1_compact), K2 (all k2_cells_phase launches of the
step) and K3c.  Usage: python tools/traffic_json.py REPORT.ncu-rep WL"""
import csv
import io
import json
import os
import subprocess
import sys

rep, wl = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
ti = h.index("gpu__time_duration.sum")
tot = {"k1": 0.0, "k2": 0.0, "k3": 0.0}
dur = {"k1": 0.0, "k2": 0.0, "k3": 0.0}
# what bounds each kernel (duration-weighted over its launches): issue slots, the L1 data pipe
# (shared-memory + global wavefronts), DRAM, resident warps -- percent of peak, ncu
LIM = {"issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "l1_data_pipe_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
       "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
       "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active"}
li = {k: h.index(v) for k, v in LIM.items() if v in h}
lim = {k: {m: 0.0 for m in li} for k in tot}
for r in rows[2:]:
    name = r[ki]
    k = "k1" if "k1_" in name else "k2" if "k2_" in name else "k3" if "k3_" in name else None
    if k is None:
        continue
    b = float(r[ri].replace(",", "")) * mult[units[ri]] + float(r[wi].replace(",", "")) * mult[units[wi]]
    tot[k] += b
    d_us = float(r[ti].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[units[ti]]
    dur[k] += d_us
    for m, i in li.items():
        lim[k][m] += float(r[i].replace(",", "")) * d_us
out = {"workload": wl, "source": os.path.relpath(rep), "dram_bytes_per_launch": {k: int(v) for k, v in tot.items()},
       "ncu_duration_us": {k: round(v, 1) for k, v in dur.items()},
       "ncu_limiters": {k: {m: round(v / dur[k], 1) for m, v in lim[k].items()} for k in tot if dur[k] > 0},
       "note": "ncu --set full, one bench step (cold caches, serialised); k2 = all tree-resident phases of the step"}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"traffic_{wl}.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out))
