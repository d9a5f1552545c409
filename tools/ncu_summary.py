"""Per-kernel summary CSV of an ncu --set full report (duration, DRAM bytes, achieved GB/s, occupancy, issue).

    python tools/ncu_summary.py report.ncu-rep out.csv [--alg name=bytes ...]
"""
import csv
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "us", 1.0), ("dram__bytes_read.sum", "dram_read_MB", 1.0),
        ("dram__bytes_write.sum", "dram_write_MB", 1.0),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct", 1.0),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1.0),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct", 1.0),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_active_pct", 1.0),
        ("sm__cycles_elapsed.avg.per_second", "sm_ghz", 1.0)]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    alg = dict(a.split("=") for a in sys.argv[3:] if "=" in a)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    head, units = rows[0], rows[1]
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel"] + [c[1] for c in COLS] + ["alg_MB", "alg_GBs"])
        for v in rows[2:]:
            d = dict(zip(head, v))
            name = d["Kernel Name"].split("(")[0].replace("void ", "")
            vals = []
            for key, _, scale in COLS:
                x = d.get(key, "")
                try:
                    vals.append(round(float(x) * scale, 4))
                except ValueError:
                    vals.append("")
            a = next((float(b) for k, b in alg.items() if k in name), None)
            us = vals[0]
            w.writerow([name] + vals + ([a, round(a / us * 1e3, 1)] if a and us else ["", ""]))   # MB/us -> GB/s


if __name__ == "__main__":
    main()
