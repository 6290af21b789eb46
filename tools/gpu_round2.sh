#!/bin/bash
# One gpurun call: GPU parity tests, smoke, both bench arms, the launch list of the bench
# command and the ncu DRAM capture of the bench's own frames.
# Usage (on the box): bash tools/gpu_round2.sh TAG [skip-tests] [skip-ncu]
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
nproc > $OUT/nproc.txt
if [ "${2:-}" != "skip-tests" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  tail -25 $OUT/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"; tail -2 $OUT/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"
tail -c 1500 $OUT/bench.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "bench ref exit $?"
tail -c 600 $OUT/bench_ref.json
if [ "${3:-}" != "skip-ncu" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $OUT/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu > /dev/null 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --nvtx --nvtx-include "bench_frames/" --clock-control none --csv --page raw \
   --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active \
   --log-file $OUT/frames.csv python tools/bench_frames.py --steps 20 > $OUT/frames.log 2>&1; echo "ncu frames exit $?"
python tools/ncu_frames.py $OUT/frames.csv 20 > $OUT/ncu_bench_frames.json 2>&1; echo "frames json exit $?"
fi
