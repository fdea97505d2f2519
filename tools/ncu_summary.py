"""Summarise an ncu report: per-kernel time, DRAM bytes, issue/FMA utilisation, stalls."""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
           "launch__grid_size"]


def main(path, min_ms=0.3):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if float(d["gpu__time_duration.sum"]) < min_ms:
            continue
        short = {"gpu__time_duration.sum": "ms", "dram__bytes_read.sum": "rdGB",
                 "dram__bytes_write.sum": "wrGB"}
        parts = []
        for m in METRICS:
            k = short.get(m, m.split("__")[1].replace("average_warps_issue_stalled_", "stall_")
                          .replace("_per_issue_active.ratio", "").replace(".avg.pct_of_peak_sustained", "%")[:22])
            parts.append(f"{k}={d.get(m, '?')}")
        print(d["Kernel Name"][:44])
        print("   " + " ".join(parts))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.3)
