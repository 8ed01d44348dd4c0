#!/bin/bash
# A/B: default libmlk vs a variant (MLK_LIB_VARIANT), cfg2 and a second config
set -u
TAG=${1:-ab}
VAR=${2:-occ5}
CFG2=${3:-cfg4}
OUT=gpurun_out
mkdir -p $OUT
for rep in 1 2; do
  timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report > $OUT/ab_${TAG}_base_$rep.json 2>&1
  MLK_LIB_VARIANT=$VAR timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report > $OUT/ab_${TAG}_${VAR}_$rep.json 2>&1
done
timeout 900 python bench.py --config $CFG2 --steps 2 --warmup 2 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report > $OUT/ab_${TAG}_base_$CFG2.json 2>&1
MLK_LIB_VARIANT=$VAR timeout 900 python bench.py --config $CFG2 --steps 2 --warmup 2 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report > $OUT/ab_${TAG}_${VAR}_$CFG2.json 2>&1
