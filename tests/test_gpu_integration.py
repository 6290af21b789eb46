"""The drop-in, linked and run.

oracle/_ref/shim_check is the UNMODIFIED reference library (compiled from
/root/reference's sources by oracle/Makefile) with its lodgs::render replaced by
integration/rasterizer_b200.cpp over liblodgs_b200.so.  The reference's own render
and CPU copies of its callers (run_bench, calibrate) stay in the binary under *_ref
names, so it checks, on the GPU box:

* a production frame (rasterizer.cpp:167-213 through the shim) against the
  reference's render: counts equal, image max-abs <= 1e-3, PSNR > 60 dB;
* a collect_kpc frame: image, pairs, kpc and BlendList bit-identical;
* the reference's calibrate (metrics.cpp:94-108), every instrumented render on the
  B200: per-view GTC, scene mean, tau and histogram bit-identical;
* the reference's bench matrix run_bench (bench.cpp:114-168) over filter (parallel /
  serial) x shrink (3 sigma / fixed / adaptive) with every render on the B200:
  FrameRow / AggregateRow fields identical to the CPU run except the timings.
"""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "oracle", "_ref", "shim_check")


def test_reference_shim_drop_in(gpu):
    if not os.path.exists(SHIM):
        pytest.fail(f"{SHIM} missing: build() compiles it where /root/reference exists")
    r = subprocess.run([SHIM], capture_output=True, text=True, timeout=600)
    line = r.stdout.strip().splitlines()[-1]
    res = json.loads(line)
    print(line)
    assert res["nodes"] == 99937 and res["n_selected"] == 86321 and res["n_pairs"] == 303131
    assert res["fast_ok"], res
    assert res["kpc_ok"], res
    assert res["calib_ok"], res
    assert res["bench_ok"], res
    assert res["bench_rows"] == 15
    assert res["max_abs"] <= 1e-3
    assert r.returncode == 0, r.stderr[-2000:]
    # the reference's own bench report (bench_json) rendered on the B200
    report = json.loads(r.stderr[r.stderr.index("{"):])
    assert [a["filter_mode"] + "/" + a["shrink_mode"] for a in report["aggregates"]] == [
        "parallel/3sigma", "parallel/fixed", "parallel/adaptive", "serial/3sigma",
        "serial/adaptive"]
    assert all(f["T_total"] > 0 for f in report["frames"])
