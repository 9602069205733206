"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export by CUDA source line."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname = "?"
hdr = None
agg, smp, src = collections.Counter(), collections.Counter(), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    key = (fname, int(r[0]))
    src[key] = r[1]
    try:
        agg[key] += float(r[ie] or 0)
        smp[key] += float(r[ss] or 0)
    except ValueError:
        pass
tot, ti = sum(smp.values()) or 1, sum(agg.values()) or 1
print(f"samples {tot:.0f}, warp instructions {ti:.0f}")
for k, v in smp.most_common(top):
    print(f"{k[0]}:{k[1]:5d} {100 * v / tot:5.1f}% stall-samples {100 * agg[k] / ti:5.1f}% inst  {src[k][:90]}")
