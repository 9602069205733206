"""Diagnostic: LLF-lambda cross on IDENTICAL inputs (oracle faces uploaded to the GPU)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import pyoracle as O
from paper_2408_03483_b200 import capi, ics

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
spec = ics.config3(n=n)
ctx = capi.Context(0)
os_ = O.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, O.CrossCfg.make(seed=1))
os_.set_state([O.round_(O.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
os_.step(1)  # some nontrivial momentum
st = os_.state()
for axis in (0, 1):
    faces_o = []
    for c in range(3):
        g = O.periodic_ghost(st[c])
        faces_o.append(O.reconstruct_faces(g, axis, spec.scheme))
    mom = 1 if axis == 0 else 2
    ops_o = [faces_o[0][0], faces_o[mom][0], faces_o[0][1], faces_o[mom][1]]
    ops_g = [ctx.tt(*t.cores()) for t in ops_o]
    cfg_o = O.CrossCfg.make(eps=1e-6, seed=1); cfg_g = capi.CrossCfg.make(eps=1e-6, seed=1)
    zo, so = O.cross(O.FN_LLF_LAMBDA, ops_o, ops_o[0], cfg_o, param=spec.g)
    zg, sg = ctx.cross(capi.FN_LLF_LAMBDA, ops_g, ops_g[0], cfg_g, param=spec.g)
    fo, fg = zo.full(), zg.full()
    print(f"axis {axis}: rank {zg.rank}/{zo.rank} sweeps {sg.sweeps}/{so.sweeps} res {sg.residual:.3e}/{so.residual:.3e} "
          f"rel diff {np.linalg.norm(fg-fo)/np.linalg.norm(fo):.3e}")
    # maxvol on the thin-Q of the guess core_y^T (the initial column choice)
    cy = ops_o[0].cores()[1]
    q, _ = np.linalg.qr(cy.T)
    print("  maxvol(guess) oracle", O.maxvol(q), " gpu", ctx.maxvol(q))
