"""Summarise an `ncu --page source --csv` (SASS) export: total instructions, top instructions by
executed count and by stall samples.  Usage: python tools/ncu_sass_top.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
body = []
for r in rows[2:]:                 # first kernel section only (a report may hold several launches)
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(h) and r[0] != "Address":
        body.append(r)
f = lambda r, k: float(r[ix[k]] or 0)
tot_i = sum(f(r, "Instructions Executed") for r in body)
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in body)
print(f"instructions executed {tot_i:.4g}, stall samples {tot_s:.4g}, sass lines {len(body)}")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(f(r, k) for r in body) for k in stalls}
print("stalls:", ", ".join(f"{k[6:]} {v:.0f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for key in ["Instructions Executed", "Warp Stall Sampling (All Samples)"]:
    print(f"--- top by {key}")
    for r in sorted(body, key=lambda r: -f(r, key))[:N]:
        print(f"{r[0]:>6} {f(r,'Instructions Executed'):>12.0f} {f(r,'Warp Stall Sampling (All Samples)'):>8.0f}  {r[1][:100]}")
