#!/bin/bash
# One gpurun call: GPU parity tests, a bench line, a launch list and an ncu --set full
# capture of the frame kernels.  Usage (on the box): bash tools/gpu_check.sh TAG [skip-tests]
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
if [ "${2:-}" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"
tail -c 3000 $OUT/bench.json
# launch list over the whole 300-frame path (skip the 30 sizing + 3 warm-up frames)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 330 -c 3000 --csv \
   --log-file $OUT/launches.csv python bench.py --steps 300 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'k_mark_internal|k_select_internal|k_filter_leaves|k_compact|k_tile_offsets' -s 15 -c 5 \
   -o $OUT/prof_filter python tools/profile_frames.py --alt 200 --frames 5 > $OUT/ncu_filter.log 2>&1; echo "ncu filter exit $?"
if [ "${3:-}" != "filter-only" ]; then
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'k_blend_ws|k_tile_sort|k_preprocess|k_emit|k_tile_offsets' -s 15 -c 6 \
   -o $OUT/prof_render python tools/profile_frames.py --alt 200 --frames 5 > $OUT/ncu_render.log 2>&1; echo "ncu render exit $?"
fi
