"""Time the device tt_from_full (ttsw_tt_from_full) on smooth dense n x n fields, host
buffers in and the TT handle out (one sync at the end), and check the reference's bound
||A - full(TT)||_F <= eps ||A||_F. Usage: python scripts/from_full_sizes.py [n ...]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2408_03483_b200 import capi  # noqa: E402

ctx = capi.Context(0)
for n in [int(a) for a in sys.argv[1:]] or [256, 512, 1024, 2048]:
    i = (np.arange(n) + 0.5) / n
    X, Y = np.meshgrid(i, i, indexing="ij")
    A = np.asfortranarray(1.0 + 0.1 * np.exp(-((X - 0.4) ** 2 + (Y - 0.6) ** 2) / 0.01)
                          + 0.05 * np.sin(6 * np.pi * (X + 0.3 * Y)))
    for eps in (1e-10,):
        ctx.from_full(A, eps)  # warm-up
        ctx.sync()
        t0 = time.perf_counter()
        t, info = ctx.from_full(A, eps, with_info=True)
        ctx.sync()
        ms = (time.perf_counter() - t0) * 1e3
        err = np.linalg.norm(t.full() - A) / np.linalg.norm(A)
        print(f"n={n} eps={eps:g} rank={t.rank} r_in={info.r_in} {ms:.1f} ms rel_err={err:.2e} ok={err <= eps}",
              flush=True)
