"""Diagnose GPU vs oracle on the MMS Dirichlet run: per-step per-component differences,
ranks, and the distance of each to the exact cell averages."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "oracle")
import mms_ref  # noqa: E402
import pyoracle as oracle  # noqa: E402
from paper_2408_03483_b200 import capi  # noqa: E402

oracle.build()
ctx = capi.Context(0)
n, tol, dt = 24, 1e-10, 0.2 / 24
ic = mms_ref.cell_averages(mms_ref.exact_conserved, n, 0.0)
variant = sys.argv[1] if len(sys.argv) > 1 else "full"
gs = capi.Solver(ctx, 1, 2, n, mms_ref.G, mms_ref.F, mms_ref.H, dt, tol, capi.CrossCfg.make(seed=1))
os_ = oracle.Solver(1, 2, n, mms_ref.G, mms_ref.F, mms_ref.H, dt, tol, oracle.CrossCfg.make(seed=1))
cores = []
for a in ic:
    u, s, vt = np.linalg.svd(a)
    k = max(1, int(np.sum(s > 1e-14 * s[0])))
    cores.append((u[:, :k] * s[:k], vt[:k]))
gs.set_state([ctx.round(ctx.tt(cx, cy), tol) for cx, cy in cores])
os_.set_state([oracle.round_(oracle.TT.from_cores(cx, cy), tol) for cx, cy in cores])


def fill(lib_ghosted):
    def f(q, t):
        st = mms_ref.ghost_strips(n, t)
        return [lib_ghosted(q[c], 1, 1, st[c][0], st[c][1], eps_tt=tol) for c in range(3)]
    return f


g_src = (lambda t: [ctx.from_full(a, tol) for a in mms_ref.cell_averages(mms_ref.mms_source, n, t)])
o_src = (lambda t: [oracle.from_full(a, tol) for a in mms_ref.cell_averages(mms_ref.mms_source, n, t)])
if variant == "nosrc":
    g_src = o_src = None
if variant == "periodic":
    gs.set_hooks(None, g_src)
    os_.set_hooks(None, o_src)
else:
    gs.set_hooks(fill(ctx.ghosted), g_src)
    os_.set_hooks(fill(oracle.ghosted), o_src)
r_g, r_o = gs.rhs(), os_.rhs()
for c in range(3):
    a, b = r_g[c].full(), r_o[c].full()
    print(f"rhs c={c} |diff|max={np.abs(a-b).max():.3e} |o|max={np.abs(b).max():.3e} ranks {r_g[c].rank} {r_o[c].rank}")
for k in range(2):
    gs.step(1)
    os_.step(1)
    ex = mms_ref.cell_averages(mms_ref.exact_conserved, n, os_.time)
    for c in range(3):
        a, b = gs.state()[c].full(), os_.state()[c].full()
        print(f"step {k} c={c} |g-o|max={np.abs(a-b).max():.3e} |o|max={np.abs(b).max():.3e} "
              f"|g-ex|={np.abs(a-ex[c]).max():.3e} |o-ex|={np.abs(b-ex[c]).max():.3e} ranks {gs.state()[c].rank} {os_.state()[c].rank}")
print("cross g", gs.cross_trace()[0][:12].tolist())
print("cross o", os_.cross_trace()[0][:12].tolist())
