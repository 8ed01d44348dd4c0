#!/bin/bash
set -u
TAG=${1:-r01g}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -k "assembly_fp64_parity or drop_phi or rank_share or cfg5_shape" > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --e2e-steps 1 --pcg-tol 0 --no-matvec-report > $OUT/bench_cfg3_$TAG.json 2> $OUT/bench_cfg3_$TAG.err
echo "bench_rc=$?" >> $OUT/bench_cfg3_$TAG.err
CUDA_LAUNCH_BLOCKING=1 MLK_TRACE=1 timeout 1500 python tools/cfg5_share.py --nranks 8 --rank 0 --out $OUT/cfg5_dbg_$TAG.json > $OUT/cfg5_dbg_$TAG.log 2>&1
echo "cfg5_rc=$?" >> $OUT/cfg5_dbg_$TAG.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> $OUT/cfg5_dbg_$TAG.log
