#!/bin/bash
set -u
TAG=${1:-r01o}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "matvec or pcg or loglik or smoke or multirank" > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench_rc=$?" >> $OUT/bench_$TAG.err
