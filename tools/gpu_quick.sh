#!/bin/bash
# Quick GPU check: smoke, GPU tests (optional -k filter), bench line.
# Usage (under gpurun): bash tools/gpu_quick.sh TAG [pytest -k expr] [bench args]
set -u
TAG=${1:-q}
KEXPR=${2:-}
BARGS=${3:-}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke_$TAG.log
if [ -n "$KEXPR" ]; then
  if [ "$KEXPR" = "all" ]; then
    timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > $OUT/pytest_$TAG.log 2>&1
  else
    timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -k "$KEXPR" > $OUT/pytest_$TAG.log 2>&1
  fi
  echo "pytest_rc=$?" >> $OUT/pytest_$TAG.log
fi
timeout 600 python bench.py --no-cpu-baseline $BARGS > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench_rc=$?" >> $OUT/bench_$TAG.err
