#!/bin/bash
# One gpurun call for a kernel experiment: selected GPU tests, the main bench line, then
# every built variant (tools/variants.sh).  Usage (on the box):
#   bash tools/gpu_quick.sh TAG "pytest -k expression" [steps]
set -u
TAG=${1:-quick}; K=${2:-}; STEPS=${3:-100}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
  tail -4 $OUT/pytest.log
fi
timeout 600 python bench.py --no-cpu --steps $STEPS --warmup 10 > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"
python -c "import json; j=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]); print('main', round(j['value'],1), {k: round(v*1e3,1) for k, v in j['stage_ms_per_frame'].items()}, {k: round(v,1) for k, v in j.get('blend_kernel_variants_fps', {}).items()})"
for d in _variants/*/; do
  [ -d "$d" ] || continue
  name=$(basename $d)
  LODGS_B200_LIB=$d/liblodgs_b200.so timeout 600 python bench.py --no-cpu --steps $STEPS --warmup 10 2>/dev/null | tail -1 > $OUT/v_$name.json
  python -c "import json; j=json.loads(open('$OUT/v_$name.json').read()); print('$name', round(j['value'],1), {k: round(v*1e3,1) for k, v in j['stage_ms_per_frame'].items()}, {k: round(v,1) for k, v in j.get('blend_kernel_variants_fps', {}).items()})"
done
