#!/bin/bash
# nested-plan scheduling change: bit-identity (hash) vs MLK_LIB_VARIANT=prev, A/B bench lines, nested tests
TAG=${1:-nest}; VAR=${2:-prev}
OUT=gpurun_out; mkdir -p $OUT
for cfg in cfg3 cfg4; do
  timeout 600 python tools/ab_hash.py $cfg >> $OUT/abhash_$TAG.txt 2>&1
  MLK_LIB_VARIANT=$VAR timeout 600 python tools/ab_hash.py $cfg >> $OUT/abhash_$TAG.txt 2>&1
done
for rep in 1 2; do
  for V in default $VAR; do
    if [ "$V" = "default" ]; then unset MLK_LIB_VARIANT; else export MLK_LIB_VARIANT=$V; fi
    for CFG in cfg4 cfg3; do
      timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
        --no-matvec-report > $OUT/ab_${TAG}_${V}_${CFG}_$rep.json 2> $OUT/ab_${TAG}_${V}_${CFG}_$rep.err
    done
  done
done
unset MLK_LIB_VARIANT
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "nested or full_size or rank" > $OUT/pytest_$TAG.log 2>&1
echo "pytest_rc=$?" >> $OUT/pytest_$TAG.log
