#!/bin/bash
# A/B/C timing: default build vs two variants (cfg2 x2 each, plus one second config)
set -u
TAG=${1:-ab3}; V1=${2}; V2=${3}; CFG2=${4:-cfg3}
OUT=gpurun_out
mkdir -p $OUT
B="python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report"
for rep in 1 2; do
  timeout 600 $B > $OUT/ab_${TAG}_base_$rep.json 2>&1
  MLK_LIB_VARIANT=$V1 timeout 600 $B > $OUT/ab_${TAG}_${V1}_$rep.json 2>&1
  MLK_LIB_VARIANT=$V2 timeout 600 $B > $OUT/ab_${TAG}_${V2}_$rep.json 2>&1
done
timeout 900 $B --config $CFG2 --steps 2 --warmup 2 > $OUT/ab_${TAG}_base_$CFG2.json 2>&1
MLK_LIB_VARIANT=$V1 timeout 900 $B --config $CFG2 --steps 2 --warmup 2 > $OUT/ab_${TAG}_${V1}_$CFG2.json 2>&1
MLK_LIB_VARIANT=$V2 timeout 900 $B --config $CFG2 --steps 2 --warmup 2 > $OUT/ab_${TAG}_${V2}_$CFG2.json 2>&1
