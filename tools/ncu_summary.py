"""Summarise an ncu report (details page) per kernel: duration, DRAM, IPC, occupancy,
dram bytes. Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread",
        "L2 Hit Rate", "No Eligible"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                                 "Metric Unit", "ID"))
    per = {}
    for r in rows[1:]:
        key = (r[ii], r[ki].split("(")[0])
        if r[mi] in WANT:
            per.setdefault(key, {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    idx = {k: h.index(k) for k in ("ID", "Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum")
           if k in h}
    units = rr[1]
    traffic = {}
    for r in rr[2:]:
        key = (r[idx["ID"]], r[idx["Kernel Name"]].split("(")[0])
        def val(k):
            v = float(r[idx[k]].replace(",", ""))
            u = units[idx[k]]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic[key] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    for key, m in per.items():
        print(f"[{key[0]}] {key[1]}: dram {traffic.get(key, 0)/1e6:.1f} MB")
        print("    " + "; ".join(f"{k}={m[k]}" for k in WANT if k in m))


if __name__ == "__main__":
    main(sys.argv[1])
