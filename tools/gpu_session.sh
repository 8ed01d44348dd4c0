#!/bin/bash
# One gpurun session: smoke, GPU tests, bench, ncu launch list, ncu full capture of K5a.
# Usage (under gpurun): bash tools/gpu_session.sh [tests|notests] [tag]
set -u
MODE=${1:-tests}
TAG=${2:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke_$TAG.log
if [ "$MODE" = "tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1
  echo "pytest_rc=$?" >> $OUT/pytest_gpu_$TAG.log
fi
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench_rc=$?" >> $OUT/bench_$TAG.err
SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report"
timeout 300 $SHORT > $OUT/short_$TAG.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $SHORT > $OUT/ncu_launch_$TAG.log 2>&1
echo "ncu_launch_rc=$?" >> $OUT/short_$TAG.log
timeout 300 $SHORT > $OUT/short2_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k k_tile_contract -s 1 -c 1 \
    -o $OUT/k5a_$TAG -f $SHORT > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu_full_rc=$?" >> $OUT/short2_$TAG.log
MLK_TRACE=1 timeout 300 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/trace_$TAG.log 2>&1
