#!/bin/bash
# ncu --set full captures of the render-side kernels at one altitude with fine
# warp-state sampling.  Usage (on the box): bash tools/gpu_prof_render.sh TAG [ALT]
OUT=gpurun_out/$1
ALT=${2:-200}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 \
   -k regex:'k_tile_offsets|k_preprocess|k_emit_keys|k_tile_sort|k_blend_ws|k_compact|k_select_internal' -s 21 -c 7 \
   -o $OUT/prof_render python tools/profile_frames.py --alt $ALT --frames 5 > $OUT/ncu_render.log 2>&1; echo "ncu render exit $?"
