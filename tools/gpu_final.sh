#!/bin/bash
# Full validation session: smoke, the whole GPU suite, default bench line (cfg4, with the oracle
# baseline), cfg3 / cfg2 lines, ncu launch list of cfg4, ncu --set full of the nested K5a and of a
# deep-level transfer launch.
set -u
TAG=${1:-r02final}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt 2>&1
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke_$TAG.log
if [ "${2:-tests}" = "tests" ]; then
  timeout 2700 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rA > $OUT/pytest_$TAG.log 2>&1
  echo "pytest_rc=$?" >> $OUT/pytest_$TAG.log
fi
timeout 1200 python bench.py > $OUT/bench_cfg4_$TAG.json 2> $OUT/bench_cfg4_$TAG.err
echo "bench_rc=$?" >> $OUT/bench_cfg4_$TAG.err
timeout 900 python bench.py --config cfg3 > $OUT/bench_cfg3_$TAG.json 2> $OUT/bench_cfg3_$TAG.err
timeout 900 python bench.py --config cfg2 > $OUT/bench_cfg2_$TAG.json 2> $OUT/bench_cfg2_$TAG.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report --config cfg4"
timeout 600 $SHORT > $OUT/short_$TAG.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_cfg4_$TAG.csv $SHORT > $OUT/ncu_launch_cfg4_$TAG.log 2>&1
echo "ncu_launch_rc=$?" >> $OUT/short_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tile_contract -s 1 -c 1 \
    -o $OUT/k5a_cfg4_$TAG -f $SHORT > $OUT/ncu_k5a_cfg4_$TAG.log 2>&1
echo "ncu_k5a_rc=$?" >> $OUT/ncu_k5a_cfg4_$TAG.log
timeout 900 ncu --set full --clock-control none -k regex:k_transfer -s 0 -c 1 \
    -o $OUT/ktr_cfg4_$TAG -f $SHORT > $OUT/ncu_ktr_cfg4_$TAG.log 2>&1
echo "ncu_ktr_rc=$?" >> $OUT/ncu_ktr_cfg4_$TAG.log
