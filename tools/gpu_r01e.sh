#!/bin/bash
# GPU suite + cfg2 bench + cfg5 rank-share dry run (reduced n) with checks.
set -u
TAG=${1:-r01e}
OUT=gpurun_out
mkdir -p $OUT
free -g > $OUT/host_mem_$TAG.txt; nproc >> $OUT/host_mem_$TAG.txt
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench_rc=$?" >> $OUT/bench_$TAG.err
timeout 900 python tools/cfg5_share.py --n 131072 --nranks 8 --rank 0 --check --out $OUT/cfg5_dry_$TAG.json > $OUT/cfg5_dry_$TAG.log 2>&1
echo "cfg5_rc=$?" >> $OUT/cfg5_dry_$TAG.log
