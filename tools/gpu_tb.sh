#!/bin/bash
# GPU tests (optionally a -k filter) + the bench line.  Usage: bash tools/gpu_tb.sh TAG [pytest -k expr]
OUT=gpurun_out/$1
mkdir -p $OUT
if [ -n "${2:-}" ]; then K="-k $2"; else K=""; fi
timeout 2400 python -m pytest tests -m gpu -q -rf $K > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
tail -4 $OUT/pytest_gpu.log
timeout 900 python bench.py --steps 100 --warmup 10 --no-cpu > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('$OUT/bench.json'))
print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'e2e_sync', round(d['e2e_sync']['value'],1), {k: round(v*1e3,1) for k,v in d['stage_ms_per_frame'].items()})"
