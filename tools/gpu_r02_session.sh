#!/bin/bash
# bench lines (auto plan) for several configs, optionally followed by the cfg5 all-ranks run
set -u
TAG=$1
CFGS=${2:-"cfg4 cfg3 cfg2"}
CFG5=${3:-no}
OUT=gpurun_out
mkdir -p $OUT
for CFG in $CFGS; do
  timeout 900 python bench.py --config $CFG --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline --pcg-tol 0 \
    > $OUT/bench_${CFG}_$TAG.json 2> $OUT/bench_${CFG}_$TAG.err
done
if [ "$CFG5" = "cfg5" ]; then
  timeout 2400 python tools/cfg5_all_ranks.py --out $OUT/cfg5_all_ranks_$TAG.json > $OUT/cfg5_all_ranks_$TAG.log 2>&1
  echo "cfg5_rc=$?" >> $OUT/cfg5_all_ranks_$TAG.log
fi
