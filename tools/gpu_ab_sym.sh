#!/bin/bash
# A/B of covsym variants: the symmetric C a parity tests per variant, then cfg3 bench lines (alternating)
TAG=$1; VARS=$2; CFG=${3:-cfg3}
OUT=gpurun_out; mkdir -p $OUT
for V in $VARS; do
  if [ "$V" = "default" ]; then unset MLK_LIB_VARIANT; else export MLK_LIB_VARIANT=$V; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "symmetric" > $OUT/pytest_${TAG}_$V.log 2>&1
  echo "pytest_rc=$?" >> $OUT/pytest_${TAG}_$V.log
done
for rep in 1 2; do
  for V in $VARS; do
    if [ "$V" = "default" ]; then unset MLK_LIB_VARIANT; else export MLK_LIB_VARIANT=$V; fi
    timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
      --no-matvec-report > $OUT/ab_${TAG}_${V}_${CFG}_$rep.json 2> $OUT/ab_${TAG}_${V}_${CFG}_$rep.err
  done
done
