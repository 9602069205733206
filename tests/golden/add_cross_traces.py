"""TEST INFRASTRUCTURE: add the oracle's per-step cross traces (rank, sweeps, pivot hash of
every TT-cross call) of the checkpoint steps to a long fixture made without them, as a
side file <fixture>_ctrace.npz (ctrace_<s> arrays). One oracle step per checkpoint.

  python tests/golden/add_cross_traces.py tests/golden/long/c3_n32.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as oracle  # noqa: E402
from paper_2408_03483_b200 import ics  # noqa: E402


def main(path):
    d = np.load(path)
    meta = eval(str(d["meta"]))
    spec = ics.config5_member(meta["member"], n=meta["n"]) if meta["config"] == "C5" else \
        ics.CONFIGS[meta["config"]](n=meta["n"])
    out = path[:-4] + "_ctrace.npz"
    have = dict(np.load(out)) if os.path.exists(out) else {}
    cks = [int(c) for c in d["checkpoints"]]
    for s0 in cks:
        key = f"ctrace_{s0}"
        if f"step_trace_{s0}" not in d or key in have or key in d:
            continue
        cfg = oracle.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank)
        o = oracle.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
        o.set_state([oracle.TT.from_cores(d[f"ck_{s0}_{c}_x"], d[f"ck_{s0}_{c}_y"]) for c in range(3)])
        o.step(1)
        tr = o.trace()[0]
        assert np.array_equal(tr[:, 4], d[f"step_trace_{s0}"][:, 1].astype(int)), s0  # same step as recorded
        have[key] = np.asarray(o.cross_trace()[0], dtype=np.int64).reshape(-1, 3)
        np.savez_compressed(out + ".tmp.npz", **have)
        os.replace(out + ".tmp.npz", out)
        print(path, s0, len(have[key]), flush=True)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
