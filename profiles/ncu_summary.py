"""Summarise an ncu --set full report (read here with `ncu -i`):
per kernel launch: time, DRAM bytes, throughput %, occupancy, L2 sectors.
Usage: python profiles/ncu_summary.py <report.ncu-rep>"""
import csv
import io
import re
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_sectors.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]


def main():
    # base units (bytes, ns, ...) for every row: with auto units each row may
    # pick its own scale while the header carries only the first row's
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    cols = [hdr.index(w) for w in WANT]
    print("kernel | " + " | ".join(f"{w} [{units[c]}]" for w, c in zip(WANT, cols)))
    for r in rows[2:]:
        m = re.search(r"(k_\w+)(<[^(]*>)?", r[ki])
        name = (m.group(1) + (m.group(2) or "")) if m else r[ki][:40]
        print(name + " | " + " | ".join(r[c] for c in cols))


if __name__ == "__main__":
    main()
