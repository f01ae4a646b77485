#!/bin/bash
set -u
O=gpurun_out/r2i; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for w in c4 sw8192 sw8192hump sw8192f32 c5 c5f32 c3 c2 c1; do
  for v in base yinl3; do
    vv=$v; [ "$v" = base ] && vv=""
    CLB_LIB_VARIANT=$vv timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}_${v}.json 2> $O/bench_${w}_${v}.err
  done
done
for w in c5 c5f32 c3; do
  CLB_CONTIG=tma timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}_xtma.json 2> $O/bench_${w}_xtma.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 6 -c 2 \
  -o $O/prof_c4 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $O/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 6 -c 2 \
  -o $O/prof_hump python bench.py --workload sw8192hump --steps 2 --warmup 3 --no-cpu > $O/ncu_hump.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_c4.csv python bench.py --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
echo done > $O/DONE
