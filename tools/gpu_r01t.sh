#!/bin/bash
set -u
TAG=${1:-r01t}
OUT=gpurun_out
mkdir -p $OUT
for cfg in cfg2 cfg4; do
  timeout 600 python tools/ab_hash.py $cfg >> $OUT/abhash_$TAG.txt 2>&1
  MLK_LIB_VARIANT=prev timeout 600 python tools/ab_hash.py $cfg >> $OUT/abhash_$TAG.txt 2>&1
done
bash tools/gpu_ab.sh $TAG prev cfg4
