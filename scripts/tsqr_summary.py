"""Summarise TTSW_PROFILE_TSQR lines: time by phase and by R bucket."""
import re, sys, collections
pat = re.compile(r"tsqr m=(\d+) n=(\d+) R=(\d+) k=(\d+) lv=(\d+)/(\d+) ms: qrx ([\d.]+) qry ([\d.]+) svd ([\d.]+) apx ([\d.]+) apy ([\d.]+)")
rows = [tuple(float(v) for v in m.groups()) for m in map(pat.search, open(sys.argv[1])) if m]
tot = [sum(r[i] for r in rows) for i in range(6, 11)]
print(f"{len(rows)} tsqr roundings, total {sum(tot):.1f} ms: qrx {tot[0]:.1f} qry {tot[1]:.1f} svd {tot[2]:.1f} apx {tot[3]:.1f} apy {tot[4]:.1f}")
b = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows:
    key = (int(r[0]), int(r[1]), min(int(r[2]) // 100 * 100, 800))
    b[key][0] += 1; b[key][1] += sum(r[6:11]); b[key][2] += r[8]
for key, (c, t, sv) in sorted(b.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"m={key[0]:6d} n={key[1]:6d} R~{key[2]:4d}+: count {c:4d} total {t:8.1f} ms (svd {sv:7.1f})")
