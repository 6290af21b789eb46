#!/bin/bash
# cfg-3 bench frames/s and cfg-4 (three-sigma) frames/s for the main build and every
# built variant (tools/variants.sh).  Usage (on the box): bash tools/gpu_cfg34.sh TAG [steps]
TAG=${1:-cfg34}; STEPS=${2:-100}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for d in main $(ls -d _variants/*/ 2>/dev/null); do
  name=$(basename $d)
  if [ "$d" != main ]; then export LODGS_B200_LIB=$d/liblodgs_b200.so; else unset LODGS_B200_LIB; fi
  timeout 600 python bench.py --no-cpu --steps $STEPS --warmup 10 2>/dev/null | tail -1 > $OUT/b_$name.json
  timeout 600 python tools/workloads.py --which cfg4 --frames 30 --three-sigma-only $WLARGS 2>/dev/null | tail -1 > $OUT/c4_$name.json
  python - <<PY
import json
b = json.loads(open("$OUT/b_$name.json").read())
c = json.loads(open("$OUT/c4_$name.json").read())
print("$name", "cfg3", round(b["value"], 1), "blend", round(b["stage_ms_per_frame"]["blend"] * 1e3, 1), "cfg4", round(c["fps"], 1))
PY
done
