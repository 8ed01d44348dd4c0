#!/bin/bash
set -u
TAG=${1:-r01n}
OUT=gpurun_out
mkdir -p $OUT
SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report"
timeout 300 $SHORT > $OUT/short_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_contract -s 0 -c 3 \
    -o $OUT/k5a3_$TAG -f $SHORT > $OUT/ncu_k5a3_$TAG.log 2>&1
echo "ncu_rc=$?" >> $OUT/ncu_k5a3_$TAG.log
