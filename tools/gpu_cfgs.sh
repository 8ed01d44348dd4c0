#!/bin/bash
# Bench lines + launch lists + K5a full captures for the larger configs.
# Usage (under gpurun): bash tools/gpu_cfgs.sh TAG "cfg3 cfg4 ..."
set -u
TAG=${1:-c}
CFGS=${2:-"cfg3 cfg4"}
OUT=gpurun_out
mkdir -p $OUT
for CFG in $CFGS; do
  timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --e2e-steps 1 --pcg-tol 0 > $OUT/bench_${CFG}_$TAG.json 2> $OUT/bench_${CFG}_$TAG.err
  echo "bench_rc=$?" >> $OUT/bench_${CFG}_$TAG.err
  SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report --config $CFG"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${CFG}_$TAG.csv $SHORT > $OUT/ncu_launch_${CFG}_$TAG.log 2>&1
  echo "ncu_launch_rc=$?" >> $OUT/ncu_launch_${CFG}_$TAG.log
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tile_contract -s 1 -c 1 \
      -o $OUT/k5a_${CFG}_$TAG -f $SHORT > $OUT/ncu_k5a_${CFG}_$TAG.log 2>&1
  echo "ncu_k5a_rc=$?" >> $OUT/ncu_k5a_${CFG}_$TAG.log
done
