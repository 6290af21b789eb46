#!/bin/bash
# Bench each built variant (tools/variants.sh): FPS and per-stage ms of the cfg-3 path.
for d in _variants/*/; do
  name=$(basename $d)
  LODGS_B200_LIB=$d/liblodgs_b200.so python bench.py --no-cpu --e2e-steps 1 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$name', round(j['value'],1), j['stage_ms_per_frame'])"
done
