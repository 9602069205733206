"""Markdown summary of the full-length parity runs (tests/test_gpu_long.py writes one JSON per
fixture under gpurun_out/long_parity/): per-step-reset rank traces and errors, the mismatch
table with margins and bands, free-run drift and end-of-run error.

  python scripts/long_parity_table.py gpurun_out/r02X/long_parity > profiles/r02_long_parity.md
"""
import glob
import json
import os
import sys


def main(d):
    print("# Full-length parity against the oracle (tests/test_gpu_long.py)\n")
    print("Per-step reset: the GPU starts every checkpoint step from the oracle's own state; "
          "`identical` = the step's whole per-rounding rank trace equals the oracle's. "
          "Free run: the GPU runs the trajectory from the same rounded IC.\n")
    print("| fixture | steps | reset steps | identical traces | worst reset err (identical) | first-mismatch hits | "
          "hits with margin ≤ 1e-6 | free run: state ranks equal (steps) | first state-rank diff | end rel L2 | worst Σh rel |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    hits_all = []
    for p in sorted(glob.glob(os.path.join(d, "*.json"))):
        t = json.load(open(p))
        if "reset" not in t:
            continue
        r = t["reset"]
        ident = sum(1 for x in r if x["identical"])
        hits = t.get("reset_hits", [])
        hits_all += [(t["fixture"], h) for h in hits]
        f = t["free"]
        end = f.get("end_rel_err")
        print(f"| {t['fixture']} | {t['steps']} | {len(r)} | {ident} | {t['reset_worst_identical_trace']:.2e} | "
              f"{len(hits)} | {sum(1 for h in hits if h.get('inside_1e-6'))} | {f['state_ranks_identical_steps']} | "
              f"{f['first_state_rank_difference']} | {end if end is None else f'{end:.2e}'} | {f['mass_rel_worst']:.1e} |")
    c2 = os.path.join(d, "c2_n1024_reset.json")
    if os.path.exists(c2):
        t = json.load(open(c2))
        errs = t["per_step_rel_err"]
        print(f"\nC2 N=1024, every one of the {t['steps']} steps restarted from the oracle's state: worst per-step "
              f"error with an identical rank trace {t['worst_identical_trace']:.2e}; max over all steps "
              f"{max(errs):.2e}; steps whose trace has a first mismatch: {len(t['hits'])}.")
        hits_all += [("c2_n1024_reset", h) for h in t["hits"]]
    if hits_all:
        print("\n## Every first rank mismatch of a reset step\n")
        print("| run | step | rounding | R | k oracle | k GPU | margin oracle | margin GPU | κ | band 4Ruκ/(0.9ε) |")
        print("|---|---|---|---|---|---|---|---|---|---|")
        for name, h in hits_all:
            print(f"| {name} | {h['step']} | {h['rounding']} | {h['r_in']} | {h['k_oracle']} | {h['k_gpu']} | "
                  f"{h['margin_oracle']:.2e} | {h['margin_gpu']:.2e} | {h['kappa']:.2e} | {h['band']:.2e} |")


if __name__ == "__main__":
    main(sys.argv[1])
