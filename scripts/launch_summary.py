"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    full = re.sub(r"^void ", "", r[ki]).split("(")[0]
    base = re.sub(r".*::", "", full)
    name = ("ttsw::" + base) if base.startswith("k_") else full
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(r[ui], 1)
    tot[name] += v
    cnt[name] += 1
ours = {k: v for k, v in tot.items() if k.startswith("ttsw::")}
T = sum(ours.values())
print(f"{'kernel':42s} {'launches':>8s} {'total ms':>10s} {'share':>6s} {'avg us':>9s}")
for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
    print(f"{k:42s} {cnt[k]:8d} {v / 1e6:10.3f} {100 * v / T:5.1f}% {v / cnt[k] / 1e3:9.2f}")
print(f"ttsw kernels: {sum(cnt[k] for k in ours)} launches, {T / 1e6:.3f} ms (non-ttsw: "
      + ", ".join(f"{k.split('<')[0][:30]} x{cnt[k]}" for k in tot if k not in ours) + ")")
