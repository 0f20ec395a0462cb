#!/bin/bash
# full validation of the committed kernel: GPU suite, smoke, all configs (fp64 and fp32), bench, launches
OUT=gpurun_out/r02r; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status
timeout 900 python tools/run_configs.py > $OUT/all_configs.jsonl 2>&1; echo "configs rc=$?" >> $OUT/status
timeout 600 python tools/run_configs.py --precision 32 > $OUT/all_configs_fp32.jsonl 2>&1; echo "configs32 rc=$?" >> $OUT/status
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?" >> $OUT/status
