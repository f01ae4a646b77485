#!/bin/bash
# the geometry pair's selector (clb_x_activity) + smoke on the final library
set -u
O=gpurun_out/r2y; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "geometry_pair or streaming_x_geometry or sw2048" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err
echo done > $O/DONE
