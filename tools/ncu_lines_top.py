"""Per-source-line instructions and stall samples of one kernel from `ncu --page source --csv
--print-source cuda,sass`.  usage: python tools/ncu_lines_top.py src.csv FUNC_SUBSTR FILE_SUBSTR [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fn, fsub = sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out, cur_f, cur_fn = [], "", ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_f = r[1]
        continue
    if len(r) == 2 and r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if fn in cur_fn and fsub in cur_f and len(r) > 8 and r[0].isdigit() and r[2] == "-":
        out.append((int(r[0]), r[1].strip()[:96], float(r[7] or 0), float(r[4] or 0)))
ti = sum(o[2] for o in out) or 1
ts = sum(o[3] for o in out) or 1
print(f"instructions {ti:.4g}  samples {ts:.4g}")
for ln, src, ins, s in sorted(out, key=lambda x: -x[3])[:top]:
    print(f"{ln:5d} {ins / 1e6:8.2f}M {100 * ins / ti:5.1f}% samp {100 * s / ts:5.1f}%  {src}")
