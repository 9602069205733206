"""One-line-per-kernel summary of `ncu --set full` reports (raw page): duration, launch
shape, DRAM traffic, throughput, FP64 pipe use and the top warp-stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = {
    "dur_us": ("gpu__time_duration.sum", 1e-3),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "cluster": ("launch__cluster_size", 1),
    "regs": ("launch__registers_per_thread", 1),
    "occ%": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "sm%": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_rd_MB": ("dram__bytes_read.sum", 1),
    "dram_wr_MB": ("dram__bytes_write.sum", 1),
    "l2hit%": ("lts__t_sector_hit_rate.pct", 1),
    "fp64%": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "dmma%": ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1),
}


def main(paths):
    print("| kernel | " + " | ".join(KEYS) + " | top stalls |")
    print("|---" * (len(KEYS) + 2) + "|")
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        for v in rows[2:]:
            d = dict(zip(h, v))
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").split("::")[-1]
            cells = []
            for key, (m, sc) in KEYS.items():
                x = d.get(m, "")
                try:
                    x = float(x.replace(",", ""))
                    u = units[h.index(m)] if m in h else ""
                    if m == "gpu__time_duration.sum":  # -> microseconds
                        x *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(u, 1.0)
                    elif u.endswith("byte"):  # -> megabytes
                        x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
                    else:
                        x *= sc
                    cells.append(f"{x:.3g}")
                except (ValueError, AttributeError):
                    cells.append("-")
            st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k] or 0) for k in h
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
            t = sum(st.values()) or 1
            top = ", ".join(f"{k} {100 * x / t:.0f}%" for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:3])
            print(f"| {name} | " + " | ".join(cells) + f" | {top} |")


if __name__ == "__main__":
    main(sys.argv[1:])
