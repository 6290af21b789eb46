#!/bin/bash
# e2e frames/s (f32 images to pinned host memory, render_batch) for the main build and every
# built variant, 3 runs each.  Usage (on the box): bash tools/e2e_probe.sh
for d in main $(ls -d _variants/*/ 2>/dev/null); do
  name=$(basename $d)
  if [ "$d" != main ]; then export LODGS_B200_LIB=$d/liblodgs_b200.so; else unset LODGS_B200_LIB; fi
  for r in 1 2 3; do
    timeout 600 python bench.py --no-cpu --steps 60 --warmup 5 2>/dev/null | tail -1 | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$name', round(j['e2e']['value'],1), round(j['e2e_sync']['value'],1), round(j['e2e_rgb8']['value'],1))"
  done
done
