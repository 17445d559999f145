"""Export a compact text summary of an .ncu-rep (per kernel: duration, DRAM
bytes, throughputs, tensor-pipe activity, occupancy) for profiles/."""
import csv
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__cluster_dim_y"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"# {rep}", "\t".join(f"{k} [{units[hdr.index(k)]}]" if k in hdr else k for k in KEYS)]
    for r in rows[2:]:
        lines.append("\t".join(r[hdr.index(k)] if k in hdr else "NA" for k in KEYS))
    return "\n".join(lines)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(summary(rep))
        print()
