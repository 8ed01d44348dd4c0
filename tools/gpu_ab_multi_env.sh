#!/bin/bash
# A/B/C... of environment settings: alternating bench lines per config, hashes per setting.
# usage: bash tools/gpu_ab_multi_env.sh TAG "cfg4 cfg3" "A:X=1" "B:MLK_LIB_VARIANT=tr1" ...
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
for spec in "$@"; do
  L=${spec%%:*}; E=${spec#*:}
  for cfg in $CFGS; do env $E timeout 600 python tools/ab_hash.py $cfg | sed "s/$/ [$L $E]/" >> $OUT/abhash_$TAG.txt 2>&1; done
done
for rep in 1 2; do
  for spec in "$@"; do
    L=${spec%%:*}; E=${spec#*:}
    for CFG in $CFGS; do
      env $E timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
        --no-matvec-report > $OUT/ab_${TAG}_${L}_${CFG}_$rep.json 2> $OUT/ab_${TAG}_${L}_${CFG}_$rep.err
    done
  done
done
