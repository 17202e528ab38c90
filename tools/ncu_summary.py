"""Per-kernel summary of an ncu --set full report (raw page csv)."""
import csv
import subprocess
import sys

STALLS = ["long_scoreboard", "barrier", "lg_throttle", "short_scoreboard", "mio_throttle", "wait",
          "math_pipe_throttle", "not_selected", "selected", "no_instruction", "membar", "drain",
          "dispatch_stall", "branch_resolving", "tex_throttle", "sleeping", "misc"]
COLS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    idx = {k: i for i, k in enumerate(h)}
    for row in r[2:]:
        name = row[idx["Kernel Name"]].split("(")[0].replace("hpsb::<unnamed>::", "")[:34]
        vals = []
        for c in COLS:
            if c in idx:
                vals.append(f"{c.split('__')[0][:4]}.{c.split('__')[1][:18]}={row[idx[c]]}{units[idx[c]][:6]}")
        st = []
        tot = 0.0
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in idx:
                try:
                    v = float(row[idx[k]])
                except ValueError:
                    continue
                tot += v
                st.append((v, s))
        st.sort(reverse=True)
        print(name, " ".join(vals))
        print("    stalls/issue:", ", ".join(f"{s}={v:.2f}" for v, s in st[:5]), f"(sum {tot:.1f})")


if __name__ == "__main__":
    main(sys.argv[1])
