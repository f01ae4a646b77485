#!/bin/bash
# strided group counting compiled only for the solvers with an x twin
set -u
O=gpurun_out/r2aa; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "golden or geometry_pair or streaming or random_configs or c5_acoustics or c3 or c4 or user" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
b() { timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu > $O/bench_$1.json 2> $O/bench_$1.err; }
for w in c5f32 c5 c3 c4 sw8192hump sw8192f32; do b $w; done
echo done > $O/DONE
