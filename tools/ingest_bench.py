"""Scene ingest timing: LDGS v1 file -> device scene.

  reference: load_scene (scene_io.cpp:213-226, incl. require_valid) in the
             native tool oracle/_ref/ref_ldgs_tool, wall time.
  device:    GpuScene.load (file -> pinned -> HBM, de-interleave + validate +
             pack kernels), wall time and its 3-phase breakdown; and
             GpuScene(tree) from host arrays (upload + device validation).
Prints one JSON line per tree.  Not a benchmark of record.

    python tools/ingest_bench.py --trees cfg3 cfg4
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import REF_LDGS_TOOL, write_ldgs  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402

TREES = {"cfg2": dict(nx=41, ny=42, depth=3), "cfg3": dict(nx=131, ny=131, depth=3),
         "cfg4": dict(nx=103, ny=104, depth=4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trees", nargs="+", default=["cfg3"])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    for name in args.trees:
        spec = TREES[name]
        tree = L.build_synthetic_tree(nx=spec["nx"], ny=spec["ny"], seed=1, depth=spec["depth"],
                                      build_seed=7)
        with tempfile.TemporaryDirectory(dir="/tmp") as d:
            path = os.path.join(d, f"{name}.ldgs")
            write_ldgs(tree, path)
            size = os.path.getsize(path)
            row = {"tree": name, "nodes": tree.node_count(), "file_bytes": size}
            if os.path.exists(REF_LDGS_TOOL):
                t0 = time.perf_counter()
                out = subprocess.run([REF_LDGS_TOOL, "load", path], capture_output=True,
                                     text=True).stdout
                row["reference_load_s"] = time.perf_counter() - t0
                row["reference_ok"] = out.startswith("OK")
            walls, phases = [], []
            for _ in range(args.reps):
                tm = np.zeros(3)
                t0 = time.perf_counter()
                s = L.GpuScene.load(path, timing_ms=tm)
                walls.append(time.perf_counter() - t0)
                phases.append(tm.copy())
                s.close()
            row["device_load_s"] = float(np.median(walls))
            ph = np.median(np.stack(phases), axis=0)
            row["device_phases_ms"] = {"read_h2d": ph[0], "deinterleave": ph[1],
                                       "validate_pack": ph[2]}
            arr = []
            for _ in range(args.reps):
                t0 = time.perf_counter()
                L.GpuScene(tree).close()
                arr.append(time.perf_counter() - t0)
            row["device_from_arrays_s"] = float(np.median(arr))
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
