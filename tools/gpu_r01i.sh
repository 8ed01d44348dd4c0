#!/bin/bash
set -u
TAG=${1:-r01i}
OUT=gpurun_out
mkdir -p $OUT
MLK_SCRATCH_BUDGET_MB=300 timeout 600 python tools/cfg5_share.py --n 131072 --stop-after-basis > $OUT/cfg5_small_budget_$TAG.log 2>&1
echo "rc=$?" >> $OUT/cfg5_small_budget_$TAG.log
MLK_SCRATCH_BUDGET_MB=300 timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/cfg5_share.py --n 131072 --stop-after-basis > $OUT/cfg5_sanitizer_$TAG.log 2>&1
echo "rc=$?" >> $OUT/cfg5_sanitizer_$TAG.log
