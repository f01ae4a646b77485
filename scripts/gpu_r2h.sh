#!/bin/bash
# step-redo variants: parity on the slow-path / random matrix, A/B bench, ncu of the default
set -u
O=gpurun_out/r2h; mkdir -p $O
for v in redo redoyinl3; do
  CLB_LIB_VARIANT=$v timeout 900 python -m pytest tests -m gpu -x -q -k "slow_path or random_configs or golden or hump or sw2048 or blowup" > $O/pytest_$v.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$v.log
done
for w in sw8192hump sw8192 c4 c5; do
  for v in base redo redoyinl3; do
    vv=$v; [ "$v" = base ] && vv=""
    CLB_LIB_VARIANT=$vv timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}_${v}.json 2> $O/bench_${w}_${v}.err
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 6 -c 2 \
  -o $O/prof_c4 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $O/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 6 -c 2 \
  -o $O/prof_hump python bench.py --workload sw8192hump --steps 2 --warmup 3 --no-cpu > $O/ncu_hump.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_c4.csv python bench.py --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
echo done > $O/DONE
