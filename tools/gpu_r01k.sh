#!/bin/bash
set -u
TAG=${1:-r01k}
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "loglik or assembly or multirank or drop_phi or rank_share or full_size or cfg5_shape" > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench_rc=$?" >> $OUT/bench_$TAG.err
MLK_TRACE=1 timeout 2400 python tools/cfg5_share.py --nranks 8 --rank 0 --check --out $OUT/cfg5_share_$TAG.json > $OUT/cfg5_share_$TAG.log 2>&1
echo "cfg5_rc=$?" >> $OUT/cfg5_share_$TAG.log
