"""Summarise an ncu report: per kernel launch, time / DRAM bytes / pipe utilisation."""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"),
        ("dram__bytes_write.sum", "dram_wr"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
        ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("launch__registers_per_thread", "regs"), ("smsp__inst_executed.sum", "warp_inst"),
        ("sm__cycles_elapsed.avg.per_second", "clk"), ("launch__grid_size", "grid")]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        vals = []
        for k, short in KEYS:
            if k in idx:
                vals.append(f"{short}={r[idx[k]]}{units[idx[k]]}")
        print(name[:60], "|", " ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
