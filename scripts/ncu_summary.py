"""Summarise an .ncu-rep: per kernel, the key throughput/pipe/stall metrics."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__occupancy_limit_registers"]
PIPES = "sm__inst_executed_pipe_"
STALL = "smsp__average_warps_issue_stalled_"


def main(path, top=12):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(h, row))
        print("=" * 100)
        print(d.get("Kernel Name", "?")[:100])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]} {units[h.index(k)]}")
        pipes = [(k, float(d[k])) for k in h if k.startswith(PIPES) and k.endswith(".avg.pct_of_peak_sustained_active")
                 and d[k] not in ("", "n/a")]
        pipes = sorted(pipes, key=lambda x: -x[1])[:8]
        print("  pipes:", ", ".join(f"{k[len(PIPES):].split('.')[0]}={v:.1f}%" for k, v in pipes))
        st = [(k, float(d[k])) for k in h if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")
              and d[k] not in ("", "n/a")]
        st = sorted(st, key=lambda x: -x[1])[:top]
        print("  stalls/issue:", ", ".join(f"{k[len(STALL):].replace('_per_issue_active.ratio','')}={v:.2f}" for k, v in st))


if __name__ == "__main__":
    main(sys.argv[1])
