"""Per-kernel mean device time and share from an ncu launch list
(--metrics gpu__time_duration.sum --csv).  Usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    d = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi:
            try:
                d[r[ki].split("(")[0].replace("void ", "")].append(
                    float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
            except ValueError:
                pass
    tot = sum(sum(v) for v in d.values())
    print(f"# {path}: {sum(len(v) for v in d.values())} launches")
    print(f"{'kernel':34s} {'n':>5s} {'mean_us':>9s} {'share':>6s}")
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        print(f"{k[:34]:34s} {len(v):5d} {sum(v) / len(v):9.2f} {sum(v) / tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
