#!/bin/bash
# Parity (full -m gpu suite or a -k subset) + bench lines of the default library.
# Usage: gpurun -- 'bash scripts/gpu_check.sh TAG "c4 sw8192" [K-expr]'
set -u
TAG=$1; WL=$2; K=${3:-}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest_gpu.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> $O/pytest_gpu.log
for w in $WL; do
  timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}.json 2> $O/bench_${w}.err
done
echo done > $O/DONE
