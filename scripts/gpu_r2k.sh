#!/bin/bash
set -u
O=gpurun_out/r2k; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for pad in 0 1 2 4; do
  CLB_PITCH_PAD=$pad timeout 400 python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu > $O/bench_c4_pad$pad.json 2> $O/bench_c4_pad$pad.err
done
CLB_LIB_VARIANT=xs4 timeout 400 python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu > $O/bench_c4_xs4.json 2> $O/bench_c4_xs4.err
for w in c5 c5f32 c3 sw8192f32 sw8192hump; do
  timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_${w}.json 2> $O/bench_${w}.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 9 -c 3 \
  -o $O/prof_c5 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu > $O/ncu_c5.log 2>&1
echo done > $O/DONE
