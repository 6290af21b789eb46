#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck / initcheck over tools/sanitize_frames.py.
# Usage (on the box): bash tools/gpu_sanitize.sh TAG
OUT=gpurun_out/$1
mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in 1 3; do
    frames=4; [ $cfg = 3 ] && frames=2
    timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_frames.py --cfg $cfg --frames $frames > $OUT/sanitize_${tool}_cfg${cfg}.log 2>&1
    echo "$tool cfg$cfg exit $?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $OUT/sanitize_${tool}_cfg${cfg}.log | tail -2 | tr '\n' ' ')"
  done
done
