"""Per-kernel summary of an ncu capture of the bench's frames (tools/bench_frames.py)
as JSON for bench.py's `traffic` / physical roofline fields:

    ncu --nvtx --nvtx-include "bench_frames/" --clock-control none --csv --page raw \
        --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__inst_issued.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,\
sm__warps_active.avg.pct_of_peak_sustained_active --log-file frames.csv \
        python tools/bench_frames.py --steps 20
    python tools/ncu_frames.py frames.csv 20 > profiles/r2_ncu_bench_frames.json
"""
import collections
import csv
import json
import sys

SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,
         "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
COLS = {"gpu__time_duration.sum": "mean_us", "dram__bytes_read.sum": "dram_rd_mb",
        "dram__bytes_write.sum": "dram_wr_mb",
        "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct"}


def main(path, frames):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    acc = collections.defaultdict(lambda: collections.defaultdict(float))
    n = collections.Counter()
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        k = r[ki].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
        n[k] += 1
        for m, name in COLS.items():
            if m in hdr:
                i = hdr.index(m)
                v = float(r[i].replace(",", ""))
                if name in ("mean_us", "dram_rd_mb", "dram_wr_mb"):
                    v *= SCALE.get(units[i], 1.0)
                acc[k][name] += v
    out = {"source": path, "frames": frames, "kernels": {}}
    for k in sorted(n, key=lambda k: -acc[k]["mean_us"]):
        d = {name: acc[k][name] / n[k] for name in acc[k]}
        d["launches"] = n[k]
        d["launches_per_frame"] = n[k] / frames
        out["kernels"][k] = d
    tot = sum(acc[k]["mean_us"] for k in n)
    for k, d in out["kernels"].items():
        d["share"] = acc[k]["mean_us"] / tot if tot else None
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
