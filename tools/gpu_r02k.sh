#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=r02k
for V in default trp8; do
  for CFG in cfg4 cfg3; do
    if [ "$V" = "default" ]; then unset MLK_LIB_VARIANT; else export MLK_LIB_VARIANT=$V; fi
    timeout 900 python bench.py --config $CFG --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
      --no-matvec-report > $OUT/ab_${TAG}_${V}_${CFG}.json 2> $OUT/ab_${TAG}_${V}_${CFG}.err
  done
done
unset MLK_LIB_VARIANT
timeout 900 python bench.py --config cfg2 --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
  --no-matvec-report > $OUT/ab_${TAG}_auto_cfg2.json 2> $OUT/ab_${TAG}_auto_cfg2.err
