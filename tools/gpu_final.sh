#!/bin/bash
# Full validation session: smoke, the whole GPU suite, default bench line (cfg4, with the oracle
# baseline), cfg3 / cfg2 lines, the reference arm, and per config an ncu launch list plus one
# ncu --set full capture of the dominant K5a launch (traffic + counters, tools/summarize_profiles.py).
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
for cfg in cfg4 cfg3 cfg2; do
  SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report --config $cfg"
  SKIP=1; [ $cfg = cfg2 ] && SKIP=0
  timeout 600 $SHORT > $OUT/short_${cfg}_$TAG.log 2>&1 && \
    timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${cfg}_$TAG.csv $SHORT > $OUT/ncu_launch_${cfg}_$TAG.log 2>&1
  echo "ncu_launch_rc=$?" >> $OUT/short_${cfg}_$TAG.log
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tile_contract -s $SKIP -c 1 \
      -o $OUT/k5a_${cfg}_$TAG -f $SHORT > $OUT/ncu_k5a_${cfg}_$TAG.log 2>&1
  echo "ncu_k5a_rc=$?" >> $OUT/ncu_k5a_${cfg}_$TAG.log
  # gpurun copies back <= 64 MiB: keep the raw page as CSV, drop the report
  ncu -i $OUT/k5a_${cfg}_$TAG.ncu-rep --page raw --csv > $OUT/k5a_${cfg}_$TAG.raw.csv 2>> $OUT/ncu_k5a_${cfg}_$TAG.log
  rm -f $OUT/k5a_${cfg}_$TAG.ncu-rep
done
du -sh $OUT
