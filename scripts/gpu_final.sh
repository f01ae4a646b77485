#!/bin/bash
# Round-end checkpoint: smoke, the full -m gpu suite, every bench line, the
# default line and the reference arm, the ncu launch list of the default
# line and full captures of the C4 and hump sweeps.
set -u
O=gpurun_out/${1:-r2final}; mkdir -p $O
{ nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv; } > $O/host.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$1.json 2> $O/bench_$1.err; }
for w in c1 c2 c3 c5 c5f32 sw8192 sw8192hump sw8192f32 c4lake; do b $w; done
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 > $O/bench_c5_full.json 2> $O/bench_c5_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_c4.csv python bench.py --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
# fp64 SW: three sweep_kernel launches per attempt (the x geometry pair + y)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 9 -c 3 \
  -o $O/prof_c4 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $O/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 9 -c 3 \
  -o $O/prof_hump python bench.py --workload sw8192hump --steps 2 --warmup 3 --no-cpu > $O/ncu_hump.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 9 -c 3 \
  -o $O/prof_c5 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu > $O/ncu_c5.log 2>&1
# summaries on the box; only the C4 report comes back (gpurun_out <= 64 MiB)
python scripts/ncu_summ.py $O/prof_c4.ncu-rep 268435456 > $O/ncu_c4.txt 2>&1
python scripts/ncu_summ.py $O/prof_hump.ncu-rep 67108864 > $O/ncu_hump.txt 2>&1
python scripts/ncu_summ.py $O/prof_c5.ncu-rep 134217728 > $O/ncu_c5.txt 2>&1
rm -f $O/prof_hump.ncu-rep $O/prof_c5.ncu-rep
du -sh $O > $O/size.txt
echo done > $O/DONE
