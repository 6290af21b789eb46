#!/bin/bash
# ncu --set full (source counters) of the blend kernels at one altitude.
# Usage (on the box): bash tools/gpu_prof_blend.sh TAG [ALT] [kernel regex]
OUT=gpurun_out/$1
ALT=${2:-200}
KR=${3:-'k_blend_tma|k_pack_blend|k_blend_wsp'}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"$KR" -s 2 -c 2 \
   -o $OUT/prof_blend python tools/profile_frames.py --alt $ALT --frames 5 > $OUT/ncu_blend.log 2>&1; echo "ncu blend exit $?"
python tools/ncu_summary.py $OUT/prof_blend.ncu-rep > $OUT/ncu_blend_summary.txt 2>&1
cat $OUT/ncu_blend_summary.txt
for k in k_blend_g4 k_blend_tma k_pack_blend k_blend_wsp; do python tools/ncu_hot.py $OUT/prof_blend.ncu-rep $k 40 > $OUT/hot_$k.txt 2>&1; done
