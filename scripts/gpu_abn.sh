#!/bin/bash
# A/B/C of several library variants: one parity subset on the default
# library, then bench lines of every variant.
# Usage: gpurun -- 'bash scripts/gpu_abn.sh TAG "base noskip inl" "sw8192 c4" [K-expr]'
set -u
TAG=$1; VARS=$2; WL=$3; K=${4:-}
O=gpurun_out/$TAG; mkdir -p $O
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
for w in $WL; do
  for v in $VARS; do
    vv=$v; [ "$v" = base ] && vv=""
    CLB_LIB_VARIANT=$vv timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}_${v}.json 2> $O/bench_${w}_${v}.err
  done
done
echo done > $O/DONE
