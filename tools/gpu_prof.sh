#!/bin/bash
# Profiling session: launch list of a short bench, ncu --set full of K5a and of the QR launches.
# Usage (under gpurun): bash tools/gpu_prof.sh TAG [config]
set -u
TAG=${1:-p}
CFG=${2:-cfg2}
OUT=gpurun_out
mkdir -p $OUT
SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report --config $CFG"
timeout 300 $SHORT > $OUT/short_$TAG.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $SHORT > $OUT/ncu_launch_$TAG.log 2>&1
echo "ncu_launch_rc=$?" >> $OUT/short_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_contract -s 1 -c 1 \
    -o $OUT/k5a_$TAG -f $SHORT > $OUT/ncu_k5a_$TAG.log 2>&1
echo "ncu_k5a_rc=$?" >> $OUT/short_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qr_wy -s 15 -c 1 \
    -o $OUT/qr_$TAG -f $SHORT > $OUT/ncu_qr_$TAG.log 2>&1
echo "ncu_qr_rc=$?" >> $OUT/short_$TAG.log
