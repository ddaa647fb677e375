"""Key metrics of every launch in an ncu --set full report (read here, no GPU).
Usage: python tools/ncu_summary.py report.ncu-rep [algorithmic_bytes_per_launch ...]"""
import csv
import io
import subprocess
import sys

WANT = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = (r[i], units[i])
        print("-" * 80)
        for k, (v, u) in d.items():
            print("%-75s %s %s" % (k, v, u))
        try:
            rd = float(d["dram__bytes_read.sum"][0].replace(",", "")) * SCALE[d["dram__bytes_read.sum"][1]]
            wr = float(d["dram__bytes_write.sum"][0].replace(",", "")) * SCALE[d["dram__bytes_write.sum"][1]]
            ms = float(d["gpu__time_duration.sum"][0].replace(",", "")) * SCALE[d["gpu__time_duration.sum"][1]]
            print("%-75s %.4g GB  (%.1f GB/s under ncu)" % ("dram traffic (read+write)", (rd + wr) / 1e9,
                                                            (rd + wr) / ms / 1e6))
        except (KeyError, ValueError):
            pass


if __name__ == "__main__":
    main()
