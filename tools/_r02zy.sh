#!/bin/bash
# final certification of HEAD (adds the SCI / XCI / MCI split; every earlier kernel SASS-identical):
# GPU suite, smoke, bench (c5 headline) and its launch list
OUT=gpurun_out/r02zy; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dedup --no-extra > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?" >> $OUT/status
