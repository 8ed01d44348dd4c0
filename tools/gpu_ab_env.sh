#!/bin/bash
# A/B of an environment switch (e.g. MLK_TR_V1=1): hash bit-identity, alternating bench lines, optional tests
# usage: bash tools/gpu_ab_env.sh TAG "ENV=VAL" "cfg4 cfg3" [pytest -k expr]
TAG=$1; ENVSET=$2; CFGS=${3:-cfg4}; KEXPR=${4:-}
OUT=gpurun_out; mkdir -p $OUT
for cfg in $CFGS; do
  timeout 600 python tools/ab_hash.py $cfg >> $OUT/abhash_$TAG.txt 2>&1
  env $ENVSET timeout 600 python tools/ab_hash.py $cfg | sed "s/$/ [$ENVSET]/" >> $OUT/abhash_$TAG.txt 2>&1
done
for rep in 1 2; do
  for V in A B; do
    for CFG in $CFGS; do
      if [ $V = A ]; then E=""; else E=$ENVSET; fi
      env $E timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
        --no-matvec-report > $OUT/ab_${TAG}_${V}_${CFG}_$rep.json 2> $OUT/ab_${TAG}_${V}_${CFG}_$rep.err
    done
  done
done
if [ -n "$KEXPR" ]; then
  timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$KEXPR" > $OUT/pytest_$TAG.log 2>&1
  echo "pytest_rc=$?" >> $OUT/pytest_$TAG.log
fi
