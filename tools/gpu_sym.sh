#!/bin/bash
# symmetric multi-vector C a: parity tests, then cfg3 / cfg4 bench lines
TAG=${1:-r02w}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "symmetric or matvec" > $OUT/pytest_sym_$TAG.log 2>&1
echo "pytest_rc=$?" >> $OUT/pytest_sym_$TAG.log
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg3_$TAG.json 2> $OUT/bench_cfg3_$TAG.err
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg4_$TAG.json 2> $OUT/bench_cfg4_$TAG.err
