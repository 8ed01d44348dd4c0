#!/bin/bash
# A/B of library variants on one config (bench lines, alternating), after a parity subset.
# Usage (under gpurun): bash tools/gpu_ab_r02.sh TAG CONFIG "variant1 variant2 ..." [pytest -k expr]
set -u
TAG=$1
CFG=$2
VARS=$3
KEXPR=${4:-}
OUT=gpurun_out
mkdir -p $OUT
if [ -n "$KEXPR" ]; then
  timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rA -k "$KEXPR" > $OUT/pytest_$TAG.log 2>&1
  echo "pytest_rc=$?" >> $OUT/pytest_$TAG.log
fi
for rep in 1 2; do
  for V in $VARS; do
    if [ "$V" = "default" ]; then unset MLK_LIB_VARIANT; else export MLK_LIB_VARIANT=$V; fi
    timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
      --no-matvec-report > $OUT/ab_${TAG}_${V}_${CFG}_$rep.json 2> $OUT/ab_${TAG}_${V}_${CFG}_$rep.err
  done
done
unset MLK_LIB_VARIANT
