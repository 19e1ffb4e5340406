"""SASS under a source-line range from `ncu -i REP --page source --csv --print-source cuda,sass`.
Usage: python tools/ncu_sass_lines.py file.csv LO HI [min_count]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
lo, hi = int(sys.argv[2]), int(sys.argv[3])
mn = float(sys.argv[4]) if len(sys.argv) > 4 else 0
cur = None
for r in rows:
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        cur = int(r[0])
        if lo <= cur <= hi:
            print(f"---- {cur}: {r[1][:100]}")
        continue
    if len(r) > 8 and r[0] == "" and r[2].startswith("0x") and cur is not None and lo <= cur <= hi:
        n = float(r[7] or 0)
        if n >= mn:
            print(f"   {n:11.0f} st {r[4]:>5}  {r[3].strip()}")
