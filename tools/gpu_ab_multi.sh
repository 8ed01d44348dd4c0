#!/bin/bash
# A/B of library variants on several configs: bash tools/gpu_ab_multi.sh TAG "cfgs" "variants"
set -u
TAG=$1
CFGS=$2
VARS=$3
OUT=gpurun_out
mkdir -p $OUT
for CFG in $CFGS; do
  for rep in 1 2; do
    for V in $VARS; do
      if [ "$V" = "default" ]; then unset MLK_LIB_VARIANT; else export MLK_LIB_VARIANT=$V; fi
      timeout 900 python bench.py --config $CFG --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
        --no-matvec-report > $OUT/ab_${TAG}_${V}_${CFG}_$rep.json 2> $OUT/ab_${TAG}_${V}_${CFG}_$rep.err
    done
  done
done
unset MLK_LIB_VARIANT
