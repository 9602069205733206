"""DRAM traffic of the rounding-class kernels over one step (fills bench.py's roofline.traffic).

Step 1 (GPU box, under ncu; only the profiled step is captured):
  ncu --profile-from-start off --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --csv --log-file gpurun_out/traffic_C4.csv python scripts/traffic.py run C4 4096 5
  (5 warm-up steps unprofiled, then one step between cudaProfilerStart/Stop; the step's
   rounding count is written to gpurun_out/traffic_C4.meta.json)
Step 2 (here): python scripts/traffic.py summarise gpurun_out/traffic_C4.csv gpurun_out/traffic_C4.meta.json \
      profiles/traffic_C4_N4096.json
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# kernels launched inside round / round_batch (tt.hpp:120-138): lazy-input gathers, CAQR and
# TSQR factorisations, the SVD of S, the Q applications
ROUND_CLASS = ("k_caqr_", "k_svd_", "k_qrcp_", "k_lq_cluster", "k_form_s_batch", "k_qr_blocks", "k_apply_blocks",
               "k_gather_jobs", "k_gather", "k_pad_copy", "k_extract_r", "k_round_small",
               "k_gemm", "k_probe_energy", "k_sumsq_part", "k_fill_identity", "k_fill_gauss")


def run(name, n, warm):
    import torch

    from paper_2408_03483_b200 import capi, ics

    spec = ics.CONFIGS[name](n=n)
    ctx = capi.Context(0)
    s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                    capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
    s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
    s.set_tracing(False)
    for _ in range(warm):
        s.step(1)
    ctx.sync()
    s.set_tracing(True)
    s.trace(clear=True)
    torch.cuda.profiler.start()
    s.step(1)
    ctx.sync()
    torch.cuda.profiler.stop()
    tr = s.trace()[0]
    m, nn, R, k = (tr[:, i].astype(float) for i in (1, 2, 3, 4))
    alg = float((8 * (m + nn) * (R + k)).sum())
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump({"config": name, "N": n, "step": warm, "roundings": int(len(tr)), "algorithmic_bytes": alg},
              open(os.path.join(ROOT, "gpurun_out", f"traffic_{name}.meta.json"), "w"))


def summarise(csv_path, meta_path, out_path):
    meta = json.load(open(meta_path))
    per = {}
    for r in csv.reader(open(csv_path)):
        if len(r) < 15 or not r[0].isdigit():
            continue
        name = r[4].split("(")[0].split("::")[-1].split("<")[0]
        d = per.setdefault(name, {"launches": set(), "dram": 0.0, "ns": 0.0})
        d["launches"].add(r[0])
        v = float(r[14].replace(",", "")) if r[14] else 0.0
        if r[12].startswith("dram__bytes"):
            d["dram"] += v
        elif r[12].startswith("gpu__time_duration"):
            d["ns"] += v
    cls = {k: v for k, v in per.items() if k.startswith(ROUND_CLASS)}
    dram = sum(v["dram"] for v in cls.values())
    out = {"config": meta["config"], "N": meta["N"], "step": meta["step"], "roundings": meta["roundings"],
           "round_class_dram_bytes": dram, "algorithmic_bytes": meta["algorithmic_bytes"],
           "traffic_over_algorithmic": dram / meta["algorithmic_bytes"] if meta["algorithmic_bytes"] else None,
           "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum over every rounding-class launch of step "
                     f"{meta['step']} (scripts/traffic.py; serialised replay, cold caches), / roundings",
           "kernels": {k: {"launches": len(v["launches"]), "dram_MB": v["dram"] / 1e6, "ms": v["ns"] / 1e6}
                       for k, v in sorted(per.items(), key=lambda kv: -kv[1]["dram"])}}
    json.dump(out, open(out_path, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("roundings", "round_class_dram_bytes", "algorithmic_bytes",
                                          "traffic_over_algorithmic")}))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    else:
        summarise(sys.argv[2], sys.argv[3], sys.argv[4])
