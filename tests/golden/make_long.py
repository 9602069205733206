"""TEST INFRASTRUCTURE: oracle trajectories for the full-length parity runs.

Runs the CPU oracle (restated reference, oracle/) for a whole BASELINE run at a reduced
grid size and writes a compact fixture the GPU tests compare against
(tests/test_gpu_long.py):

* ``ranks``      (steps+1, 3)  state ranks after every step (row 0 = the rounded IC);
* ``ktrace``     int32 (rows, 4)  every rounding of every step: step, r_in, k_out, crosses before;
* ``near``       rows of ``ktrace`` whose truncation margin |m| < 1e-2, with margin and kappa
                 (the only decisions a roundoff-level input change can flip);
* ``mass``       (steps+1,)  sum of h after every step;
* ``ck_<s>_<c>_x|y``  state cores at the checkpoint steps (every ``--every`` steps, the step
                 after each, and the last), so a GPU run can be compared along the trajectory
                 and re-started from the oracle's own state for per-step tests;
* ``step_trace_<s>``  full rounding trace (k, margin, kappa) of the steps s -> s+1 whose
                 start state is a checkpoint (the per-step-reset rank comparison);
* ``ctrace_<s>``  the cross calls of those steps (rank, sweeps, pivot hash): where the
                 GPU's pivots first differ (a tie split), later decisions see other inputs
                 (tests/golden/add_cross_traces.py adds them to fixtures made without).

  python tests/golden/make_long.py C3 32 1000 --every 100 --out tests/golden/long/c3_n32.npz
  python tests/golden/make_long.py C5 32 500 --member 3 --every 100 --out ...

The file is written every ``--every`` steps, so a partial run is usable. Follows the
reference time loop run_impl (proj/src/harness.cpp:104-139) with a fixed EpsSchedule.
"""
import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as oracle  # noqa: E402
from paper_2408_03483_b200 import ics  # noqa: E402


def spec_for(name, n, member):
    if name == "C5":
        return ics.config5_member(member, n=n)
    return ics.CONFIGS[name](n=n)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("config")
    p.add_argument("n", type=int)
    p.add_argument("steps", type=int)
    p.add_argument("--member", type=int, default=0)
    p.add_argument("--every", type=int, default=100)
    p.add_argument("--extra", default="", help="comma-separated extra checkpoint steps")
    p.add_argument("--out", required=True)
    a = p.parse_args()
    spec = spec_for(a.config, a.n, a.member)
    cfg = oracle.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank)
    s = oracle.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
    s.set_state([oracle.round_(oracle.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
    ck = set(range(0, a.steps + 1, a.every)) | {a.steps}
    ck |= {c + 1 for c in list(ck) if c + 1 <= a.steps}
    ck |= {int(x) for x in a.extra.split(",") if x}
    ranks = [[t.rank for t in s.state()]]
    mass = [s.state()[0].cores()[0].sum(axis=0) @ s.state()[0].cores()[1].sum(axis=1)]
    kt, near = [], []
    arrays = {}

    def save_state(step):
        for c, t in enumerate(s.state()):
            cx, cy = t.cores()
            arrays[f"ck_{step}_{c}_x"] = cx
            arrays[f"ck_{step}_{c}_y"] = cy

    def flush(done):
        meta = dict(config=a.config, n=a.n, member=a.member, steps_done=done, steps=a.steps,
                    tol=spec.tol, dt=spec.dt)
        tmp = a.out + ".tmp.npz"
        np.savez_compressed(tmp, ranks=np.array(ranks, dtype=np.int32), mass=np.array(mass),
                            ktrace=np.array(kt, dtype=np.int32).reshape(-1, 4),
                            near=np.array(near, dtype=np.float64).reshape(-1, 5),
                            checkpoints=np.array(sorted(c for c in ck if c <= done), dtype=np.int32),
                            meta=np.array(repr(meta)), **arrays)
        os.replace(tmp, a.out)

    save_state(0)
    t0 = time.time()
    for k in range(a.steps):
        s.step(1)
        tr, mg, ka = s.trace()
        ct, cres = s.cross_trace()
        for i in range(len(tr)):
            kt.append((k, tr[i, 3], tr[i, 4], tr[i, 5]))
            if abs(mg[i]) < 1e-2:
                near.append((k, i, tr[i, 4], mg[i], ka[i]))
        if k in ck:  # the step that starts at checkpoint k
            arrays[f"step_trace_{k}"] = np.column_stack([tr[:, 3], tr[:, 4], tr[:, 5], mg, ka])
            arrays[f"ctrace_{k}"] = np.asarray(ct, dtype=np.int64).reshape(-1, 3)  # rank, sweeps, pivot hash
        st = s.state()
        ranks.append([t.rank for t in st])
        hx, hy = st[0].cores()
        mass.append(hx.sum(axis=0) @ hy.sum(axis=1))
        if k + 1 in ck:
            save_state(k + 1)
        if (k + 1) % a.every == 0 or k + 1 == a.steps:
            flush(k + 1)
            print(f"{a.config} n={a.n} m={a.member}: step {k + 1}/{a.steps} ranks {ranks[-1]} "
                  f"{time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
