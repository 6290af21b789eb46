#!/bin/bash
# ncu --set full (source counters) of the non-blend frame kernels at one altitude.
# Usage (on the box): bash tools/gpu_prof_stages.sh TAG [ALT]
OUT=gpurun_out/$1
ALT=${2:-200}
mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --import-source on \
   -k regex:'k_preprocess|k_emit_keys|k_tile_sort|k_tile_offsets|k_mark_internal|k_filter_leaves|k_select_internal|k_compact' -s 16 -c 8 \
   -o $OUT/prof_stages python tools/profile_frames.py --alt $ALT --frames 4 > $OUT/ncu_stages.log 2>&1; echo "ncu exit $?"
python tools/ncu_summary.py $OUT/prof_stages.ncu-rep > $OUT/ncu_stages_summary.txt 2>&1
cat $OUT/ncu_stages_summary.txt
for k in k_preprocess k_emit_keys k_tile_sort k_mark_internal k_filter_leaves; do python tools/ncu_hot.py $OUT/prof_stages.ncu-rep $k 40 > $OUT/hot_$k.txt 2>&1; done
