"""Top SASS lines of one kernel in an ncu report by stall samples.
Usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [N]"""
import csv
import io
import subprocess
import sys


def main(path, kern, n=25):
    out = subprocess.run(["ncu", "-i", path, "-k", kern, "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    si, ie, te, ws, wn = (hdr.index(k) for k in ("Source", "Instructions Executed",
                                                  "Thread Instructions Executed",
                                                  "Warp Stall Sampling (All Samples)",
                                                  "Warp Stall Sampling (Not-issued Samples)"))
    data, tot_i, tot_w = [], 0, 0
    for i, r in enumerate(rows[2:]):
        try:
            ni, nw = int(r[ie]), int(r[ws] or 0)
        except (ValueError, IndexError):
            continue
        tot_i += ni
        tot_w += nw
        data.append((nw, i, ni, int(r[te] or 0), r[si].strip()[:70]))
    print(f"{kern}: warp instr {tot_i}, stall samples {tot_w}")
    for d in sorted(data, reverse=True)[:n]:
        avg = d[3] / d[2] if d[2] else 0
        print(f"  {d[0]:6d} @{d[1]:4d} inst={d[2]:10d} thr/inst={avg:5.1f}  {d[4]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
