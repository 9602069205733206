"""Summarise TTSW_PROFILE_TSQR 'caqr group' lines: time by phase, group size and R bucket."""
import re, sys, collections
pat = re.compile(r"caqr group (\d+)/(\d+) m=(\d+) n=(\d+) R=(\d+) k=(\d+) ms: qr ([\d.]+) svd ([\d.]+) apply ([\d.]+)")
rows = [m.groups() for m in map(pat.search, open(sys.argv[1])) if m]
tot = [0.0, 0.0, 0.0]
by_size = collections.Counter()
byR = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for r in rows:
    i, nb, m, n, R, k = map(int, r[:6])
    q, s, a = map(float, r[6:])
    tot[0] += q; tot[1] += s; tot[2] += a
    if i == 0: by_size[nb] += 1
    b = byR[min(R // 100 * 100, 800)]
    b[0] += 1; b[1] += q; b[2] += s; b[3] += a
print(f"{len(rows)} CAQR roundings, {sum(by_size.values())} groups, sizes {dict(by_size)}; total {sum(tot):.1f} ms: qr {tot[0]:.1f} svd {tot[1]:.1f} apply {tot[2]:.1f}")
for R, (c, q, s, a) in sorted(byR.items()):
    print(f"  R~{R:4d}+: {c:4d} roundings, qr {q:8.1f} svd {s:8.1f} apply {a:8.1f} ms")
