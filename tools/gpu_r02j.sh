#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=r02j
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rA -x -k "nested_and_direct or full_size_blocks and cfg3" > $OUT/pytest_$TAG.log 2>&1
echo "pytest_rc=$?" >> $OUT/pytest_$TAG.log
for V in default trminb2; do
  for CFG in cfg4 cfg3; do
    if [ "$V" = "default" ]; then unset MLK_LIB_VARIANT; else export MLK_LIB_VARIANT=$V; fi
    timeout 900 python bench.py --config $CFG --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
      --no-matvec-report > $OUT/ab_${TAG}_${V}_${CFG}.json 2> $OUT/ab_${TAG}_${V}_${CFG}.err
  done
done
unset MLK_LIB_VARIANT
timeout 900 python bench.py --config cfg2 --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
  --no-matvec-report > $OUT/ab_${TAG}_auto_cfg2.json 2> $OUT/ab_${TAG}_auto_cfg2.err
MLK_ASSEMBLY=nested timeout 900 python bench.py --config cfg2 --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 \
  --no-matvec-report > $OUT/ab_${TAG}_nested_cfg2.json 2> $OUT/ab_${TAG}_nested_cfg2.err
SHORT="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --no-matvec-report --config cfg4"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tile_contract -s 1 -c 1 \
    -o $OUT/k5n_cfg4_$TAG -f $SHORT > $OUT/ncu_k5n_cfg4_$TAG.log 2>&1
echo "ncu_rc=$?" >> $OUT/ncu_k5n_cfg4_$TAG.log
timeout 900 ncu --set full --clock-control none -k regex:k_transfer -s 8 -c 1 \
    -o $OUT/ktr_cfg4_$TAG -f $SHORT > $OUT/ncu_ktr_cfg4_$TAG.log 2>&1
echo "ncu_rc=$?" >> $OUT/ncu_ktr_cfg4_$TAG.log
