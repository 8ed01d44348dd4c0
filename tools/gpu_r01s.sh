#!/bin/bash
set -u
TAG=${1:-r01s}
OUT=gpurun_out
mkdir -p $OUT
for cfg in cfg2 cfg3; do
  timeout 600 python tools/ab_hash.py $cfg >> $OUT/abhash_$TAG.txt 2>&1
  MLK_LIB_VARIANT=prev timeout 600 python tools/ab_hash.py $cfg >> $OUT/abhash_$TAG.txt 2>&1
done
bash tools/gpu_ab.sh $TAG prev cfg3
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "matvec or assembly or identity or smoke or pcg" > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?" >> $OUT/pytest_gpu_$TAG.log
