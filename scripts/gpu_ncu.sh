#!/bin/bash
# ncu evidence: launch list of the default bench (C4) and a --set full capture
# of one x and one y sweep of WORKLOAD.  Usage: gpurun -- 'bash scripts/gpu_ncu.sh TAG WORKLOAD [pytest -k expr]'
set -u
TAG=$1; W=${2:-c4}; K=${3:-}
O=gpurun_out/$TAG; mkdir -p $O
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_$W.csv python bench.py --workload $W --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|sweep_contig" -s 6 -c 2 \
  -o $O/prof_$W python bench.py --workload $W --steps 2 --warmup 3 --no-cpu > $O/ncu_$W.log 2>&1
echo done > $O/DONE
