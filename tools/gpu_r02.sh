#!/bin/bash
# Round-2 GPU session: smoke, GPU tests (-k filter or "all"), default bench line, ncu launch list
# of a short bench, ncu --set full of one K5a launch.
# Usage (under gpurun): bash tools/gpu_r02.sh TAG [pytest -k expr|all|none] [config] [bench|nobench] [ncu|noncu]
set -u
TAG=${1:-r02}
KEXPR=${2:-none}
CFG=${3:-cfg4}
DOBENCH=${4:-bench}
DONCU=${5:-ncu}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt 2>&1
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke_$TAG.log
if [ "$KEXPR" = "all" ]; then
  timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rA > $OUT/pytest_$TAG.log 2>&1
  echo "pytest_rc=$?" >> $OUT/pytest_$TAG.log
elif [ "$KEXPR" != "none" ]; then
  timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rA -k "$KEXPR" > $OUT/pytest_$TAG.log 2>&1
  echo "pytest_rc=$?" >> $OUT/pytest_$TAG.log
fi
if [ "$DOBENCH" = "bench" ]; then
  timeout 900 python bench.py --config $CFG > $OUT/bench_${CFG}_$TAG.json 2> $OUT/bench_${CFG}_$TAG.err
  echo "bench_rc=$?" >> $OUT/bench_${CFG}_$TAG.err
fi
if [ "$DONCU" = "ncu" ]; then
  SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report --config $CFG"
  timeout 600 $SHORT > $OUT/short_${CFG}_$TAG.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${CFG}_$TAG.csv $SHORT > $OUT/ncu_launch_${CFG}_$TAG.log 2>&1
  echo "ncu_launch_rc=$?" >> $OUT/short_${CFG}_$TAG.log
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_tile_contract -s 1 -c 1 \
      -o $OUT/k5a_${CFG}_$TAG -f $SHORT > $OUT/ncu_k5a_${CFG}_$TAG.log 2>&1
  echo "ncu_k5a_rc=$?" >> $OUT/short_${CFG}_$TAG.log
fi
