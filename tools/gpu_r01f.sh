#!/bin/bash
# GPU suite, cfg2/cfg3/cfg4 bench lines, cfg5 full-size rank-0-of-8 share with checks.
set -u
TAG=${1:-r01f}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench_rc=$?" >> $OUT/bench_$TAG.err
for CFG in cfg3 cfg4; do
  timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --e2e-steps 1 --pcg-tol 0 > $OUT/bench_${CFG}_$TAG.json 2> $OUT/bench_${CFG}_$TAG.err
  echo "bench_rc=$?" >> $OUT/bench_${CFG}_$TAG.err
done
timeout 1800 python tools/cfg5_share.py --nranks 8 --rank 0 --check --out $OUT/cfg5_share_$TAG.json > $OUT/cfg5_share_$TAG.log 2>&1
echo "cfg5_rc=$?" >> $OUT/cfg5_share_$TAG.log
