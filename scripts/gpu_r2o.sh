#!/bin/bash
set -u
O=gpurun_out/r2o; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
CLB_LIB_VARIANT=x128 timeout 900 python -m pytest tests -m gpu -x -q -k "golden or random_configs or sw2048 or segmentation" > $O/pytest_x128.log 2>&1; echo "pytest rc=$?" >> $O/pytest_x128.log
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
for w in c4 c4lake sw8192 sw8192hump; do CLB_LIB_VARIANT=x128 b $w ${w}_x128; done
for w in c1 c2 c3 c4 c5 c5f32 sw8192 sw8192hump sw8192f32 c4lake; do b $w $w; done
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_c4.csv python bench.py --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 9 -c 3 \
  -o $O/prof_c5 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu > $O/ncu_c5.log 2>&1
echo done > $O/DONE
