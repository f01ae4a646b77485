#!/bin/bash
set -u
O=gpurun_out/r2l; mkdir -p $O
CLB_LIB_VARIANT=xm4 timeout 900 python -m pytest tests -m gpu -x -q -k "golden or random_configs or c5 or segmentation" > $O/pytest_xm4.log 2>&1; echo "pytest rc=$?" >> $O/pytest_xm4.log
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
for w in c5 c5f32; do
  b $w ${w}_base
  CLB_LIB_VARIANT=xm4 b $w ${w}_xm4
  CLB_TMA_PROMO=64 b $w ${w}_promo64
  CLB_TMA_PROMO=0 b $w ${w}_promo0
  CLB_LIB_VARIANT=xm4 CLB_TMA_PROMO=64 b $w ${w}_xm4promo64
done
b c4 c4_base
CLB_TMA_PROMO=256 b c4 c4_promo256
CLB_TMA_PROMO=64 b c4 c4_promo64
CLB_LIB_VARIANT=nostore b c4 c4_nostore
b sw8192hump hump_base
echo done > $O/DONE
