"""Per-source-line warp-instruction totals of one kernel from
`ncu -i REP --page source --csv --kernel-name K --print-source cuda,sass > file.csv`.
Usage: python tools/ncu_lines.py file.csv [N] [lo-hi ...]   (top-N lines; optional line ranges summed)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
per, src, stall = {}, {}, {}
for r in rows:
    if len(r) > 8 and r[0] and r[0] != "Line No" and r[0].isdigit() and r[2] == "-":
        ln = int(r[0])
        try:
            per[ln] = per.get(ln, 0) + float(r[7] or 0)
            stall[ln] = stall.get(ln, 0) + float(r[4] or 0)
        except ValueError:
            continue
        src[ln] = r[1]
tot = sum(per.values())
print(f"total warp instructions {tot:.4g}")
for ln, v in sorted(per.items(), key=lambda x: -x[1])[:N]:
    print(f"{ln:5d} {v:12.0f} {100*v/tot:5.1f}%  stall {stall[ln]:7.0f}  {src.get(ln,'')[:80]}")
for rg in sys.argv[3:]:
    a, b = map(int, rg.split("-"))
    v = sum(x for l, x in per.items() if a <= l <= b)
    print(f"lines {a}-{b}: {v:.4g} ({100*v/tot:.1f}%)")
