"""Per-source-line stall samples from `ncu -i X.ncu-rep --page source --print-source cuda,sass --csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
lines = []
for r in rows:
    if len(r) >= 8 and r[0].isdigit() and r[2] == "-":
        lines.append((int(r[0]), r[1], int(r[4] or 0), int(r[7] or 0)))
tot = sum(l[2] for l in lines)
print("total samples", tot)
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for ln, src, smp, inst in lines:
    if smp > thr * tot:
        print(f"{100 * smp / tot:5.1f}%  line {ln:4d}  inst {inst:9d} | {src[:120]}")
