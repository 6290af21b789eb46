"""Summarise an ncu --set full report per kernel launch: duration, DRAM bytes read/written,
DRAM and SM throughput, registers, achieved occupancy, issue-slot utilisation.

    python tools/ncu_summary.py report.ncu-rep [> profiles/rNN_ncu_full.txt]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
]

SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,
         "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          ",".join(m for m, _ in METRICS)], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    cols = [(hdr.index(m), name) for m, name in METRICS if m in hdr]
    print(f"# {path}")
    print("# dram_rd/dram_wr in MB per launch (cold caches: ncu flushes before each replay)")
    print("kernel".ljust(34) + "".join(name.rjust(9) for _, name in cols))
    for r in rows[2:]:
        vals = []
        for i, name in cols:
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                vals.append("-".rjust(9))
                continue
            v *= SCALE.get(units[i], 1.0) if name in ("us", "dram_rd", "dram_wr") else 1.0
            vals.append(f"{v:9.2f}")
        print(r[ki].split("(")[0].replace("void ", "")[:34].ljust(34) + "".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
