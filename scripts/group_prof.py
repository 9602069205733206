"""Aggregate the TTSW_PROFILE_TSQR / TTSW_PROFILE_RHS stderr of scripts/time_step.py: the CAQR-path
rounding groups of the last step (three rhs), largest first."""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
idx = [i for i, l in enumerate(lines) if l.startswith("rhs ghost")]
seg = lines[idx[-nrhs]:]
groups = []
pat = re.compile(r"caqr group (\d+)/(\d+) m=(\d+) n=(\d+) R=(\d+) k=(\d+) sketch=(-?\d+) ms: qr ([\d.]+) svd ([\d.]+) apply ([\d.]+)")
for l in seg:
    m = pat.match(l)
    if m:
        i, nb, mm, nn, R, k, sk = map(int, m.groups()[:7])
        qr, svd, ap = map(float, m.groups()[7:])
        if i == 0:
            groups.append({"nb": nb, "R": [], "k": [], "sk": [], "qr": qr * nb, "svd": svd * nb, "apply": ap * nb, "m": mm, "n": nn})
        groups[-1]["R"].append(R)
        groups[-1]["k"].append(k)
        groups[-1]["sk"].append(sk)
    elif l.startswith("rhs ") or l.startswith("phys "):
        print(l)
print(len(groups), "CAQR groups in the last step")
for g in sorted(groups, key=lambda g: -(g["qr"] + g["svd"] + g["apply"]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    t = g["qr"] + g["svd"] + g["apply"]
    print(f"nb={g['nb']:2d} m={g['m']} n={g['n']} R={g['R']} k={g['k']} sketch={g['sk']} qr {g['qr']:.2f} svd {g['svd']:.2f} apply {g['apply']:.2f} tot {t:.2f}")
print("sum qr %.1f svd %.1f apply %.1f" % tuple(sum(g[x] for g in groups) for x in ("qr", "svd", "apply")))
