#!/bin/bash
# GPU tests + racecheck + bench (no ncu).  Usage (on the box): bash tools/gpu_round2b.sh TAG
set -u
OUT=gpurun_out/$1
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
tail -14 $OUT/pytest_gpu.log
for cfg in 1 3; do
  frames=4; [ $cfg = 3 ] && frames=2
  timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_frames.py --cfg $cfg --frames $frames > $OUT/sanitize_racecheck_cfg${cfg}.log 2>&1
  echo "racecheck cfg$cfg exit $?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/sanitize_racecheck_cfg${cfg}.log | tail -1)"
done
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"
./oracle/_ref/shim_check > $OUT/shim_check.json 2> $OUT/shim_bench_report.json; echo "shim exit $?"; cat $OUT/shim_check.json
