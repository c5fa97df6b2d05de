"""Summarise an .ncu-rep (raw page) into the metrics the roofline needs."""
import csv
import subprocess
import sys

WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    units = rows[1]
    for r in rows[2:]:
        print("---")
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w}: {r[i][:100]} {units[i]}")
        if "dram__bytes_read.sum" in h:
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
                     "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}

            def val(name):
                i = h.index(name)
                return float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
            t = val("gpu__time_duration.sum")
            b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            print(f"  => DRAM GB/s (traffic/duration): {b / t / 1e9:.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
