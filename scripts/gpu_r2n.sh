#!/bin/bash
set -u
O=gpurun_out/r2n; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "golden or random_configs or c4 or sw2048 or slow_path or blowup or hump" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$2.json 2> $O/bench_$2.err; }
b c4lake c4lake
b c4 c4
b sw8192 sw8192
b sw8192f32 sw8192f32
b sw8192hump hump
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 6 -c 2 \
  -o $O/prof_lake python bench.py --workload c4lake --steps 2 --warmup 3 --no-cpu > $O/ncu_lake.log 2>&1
echo done > $O/DONE
