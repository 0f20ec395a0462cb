#!/bin/bash
# last full GPU suite + smoke of the round on HEAD (as the driver runs them)
OUT=gpurun_out/r02zze; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo "build rc=$?" >> $OUT/status
timeout 1500 python -m pytest tests/ -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status
timeout 600 python bench.py --steps 3 --warmup 3 > $OUT/bench_short.json 2> $OUT/bench_short.err; echo "bench rc=$?" >> $OUT/status
