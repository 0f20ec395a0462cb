#!/bin/bash
OUT=gpurun_out/r02x; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status
timeout 900 python tools/perf_variants.py build_variants/lib_grp4.so paper_2412_11614_b200/libisrs_egn.so --config=c5 --coi=100 --reps=3 > $OUT/variants.txt 2>&1
timeout 900 python bench.py --no-cpu > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status
