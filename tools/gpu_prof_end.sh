set -u
OUT=gpurun_out; TAG=r02end; cfg=cfg4
SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report --config $cfg"
timeout 600 $SHORT > $OUT/short_${cfg}_$TAG.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_${cfg}_$TAG.csv $SHORT > $OUT/ncu_launch_${cfg}_$TAG.log 2>&1
echo "ncu_launch_rc=$?" >> $OUT/short_${cfg}_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tile_contract -s 1 -c 1 \
    -o $OUT/k5a_${cfg}_$TAG -f $SHORT > $OUT/ncu_k5a_${cfg}_$TAG.log 2>&1
echo "ncu_k5a_rc=$?" >> $OUT/ncu_k5a_${cfg}_$TAG.log
ncu -i $OUT/k5a_${cfg}_$TAG.ncu-rep --page raw --csv > $OUT/k5a_${cfg}_$TAG.raw.csv 2>> $OUT/ncu_k5a_${cfg}_$TAG.log
rm -f $OUT/k5a_${cfg}_$TAG.ncu-rep
