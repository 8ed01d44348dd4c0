#!/bin/bash
# A/B timing against the MLK_LIB_VARIANT build, then a GPU test subset (-k expression)
set -u
TAG=${1:-abt}
VAR=${2:-prev}
CFG2=${3:-cfg3}
KEXPR=${4:-matvec}
OUT=gpurun_out
mkdir -p $OUT
bash tools/gpu_ab.sh $TAG $VAR $CFG2
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "$KEXPR" > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?" >> $OUT/pytest_gpu_$TAG.log
