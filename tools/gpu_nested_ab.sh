#!/bin/bash
# nested vs direct assembly: parity subset, then bench lines per config and mode
set -u
TAG=$1
CFGS=${2:-"cfg4 cfg3 cfg2"}
KEXPR=${3:-}
OUT=gpurun_out
mkdir -p $OUT
if [ -n "$KEXPR" ]; then
  timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rA -x -k "$KEXPR" > $OUT/pytest_$TAG.log 2>&1
  echo "pytest_rc=$?" >> $OUT/pytest_$TAG.log
fi
for CFG in $CFGS; do
  for MODE in nested direct; do
    MLK_ASSEMBLY=$MODE timeout 900 python bench.py --config $CFG --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline \
      --pcg-tol 0 --no-matvec-report > $OUT/ab_${TAG}_${MODE}_${CFG}.json 2> $OUT/ab_${TAG}_${MODE}_${CFG}.err
  done
done
