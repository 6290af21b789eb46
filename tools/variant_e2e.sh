#!/bin/bash
# e2e (f32 and 8-bit) frames/s of each built variant (tools/variants.sh) on the cfg-3 path.
for d in _variants/*/; do
  name=$(basename $d)
  LODGS_B200_LIB=$d/liblodgs_b200.so timeout 300 python bench.py --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$name', round(j['value'],1), round(j['e2e']['value'],1), round(j['e2e_rgb8']['value'],1))"
done
