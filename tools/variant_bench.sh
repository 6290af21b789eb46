#!/bin/bash
# Bench each built variant (tools/variants.sh): frames/s and per-stage ms of the cfg-3 path.
# Usage (on the box): bash tools/variant_bench.sh [steps]
STEPS=${1:-100}
for d in _variants/*/; do
  name=$(basename $d)
  LODGS_B200_LIB=$d/liblodgs_b200.so python bench.py --no-cpu --steps $STEPS --warmup 10 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$name', round(j['value'],1), 'e2e', round(j['e2e']['value'],1), {k: round(v*1e3,1) for k, v in j['stage_ms_per_frame'].items()})"
done
