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
for r in rows[2:]:
    name = r[ki]
    k = "k1" if "k1_" in name else "k2" if "k2_" in name else "k3" if "k3_" in name else None
    if k is None:
        continue
    b = float(r[ri].replace(",", "")) * mult[units[ri]] + float(r[wi].replace(",", "")) * mult[units[wi]]
    tot[k] += b
    dur[k] += float(r[ti].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[units[ti]]
out = {"workload": wl, "source": os.path.relpath(rep), "dram_bytes_per_launch": {k: int(v) for k, v in tot.items()},
       "ncu_duration_us": {k: round(v, 1) for k, v in dur.items()},
       "note": "ncu --set full, one bench step (cold caches, serialised); k2 = all tree-resident phases of the step"}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"traffic_{wl}.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out))
