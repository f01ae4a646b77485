#!/bin/bash
# A/B of a library variant: its parity subset, then bench lines of both.
# Usage: gpurun -- 'bash scripts/gpu_ab.sh TAG VARIANT "sw8192 c5" [K-expr]'
set -u
TAG=$1; VAR=$2; WL=$3; K=${4:-"golden or random_configs or slow_path or segmentation or sw2048"}
O=gpurun_out/$TAG; mkdir -p $O
CLB_LIB_VARIANT=$VAR timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest_$VAR.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$VAR.log
for w in $WL; do
  for v in "" $VAR; do
    CLB_LIB_VARIANT=$v timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}_${v:-base}.json 2> $O/bench_${w}_${v:-base}.err
  done
done
echo done > $O/DONE
