#!/bin/bash
# bit-identity (hash) + A/B timing against MLK_LIB_VARIANT, then a GPU test subset
set -u
TAG=${1:-abh}
VAR=${2:-prev}
CFG2=${3:-cfg3}
KEXPR=${4:-basis}
OUT=gpurun_out
mkdir -p $OUT
for cfg in cfg2 $CFG2; do
  timeout 600 python tools/ab_hash.py $cfg >> $OUT/abhash_$TAG.txt 2>&1
  MLK_LIB_VARIANT=$VAR timeout 600 python tools/ab_hash.py $cfg >> $OUT/abhash_$TAG.txt 2>&1
done
bash tools/gpu_abtest.sh $TAG $VAR $CFG2 "$KEXPR"
