#!/bin/bash
# MODE_SEGWP (warp-private envelope rows, no CTA barrier in the span loop) vs the CTA-wide table:
# c4 timing (3 COIs and all 80), then the GPU parity subset on the new default
OUT=gpurun_out/r02zp; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 600 python tools/perf_variants.py build_variants/lib_wp0.so build_variants/lib_wp1.so build_variants/lib_wp0.so build_variants/lib_wp1.so --config=c4 --coi=0,40,79 --reps=3 >> $OUT/variants.txt 2>&1
timeout 600 python tools/perf_variants.py build_variants/lib_wp0.so build_variants/lib_wp1.so --config=c4 --reps=2 >> $OUT/variants.txt 2>&1
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "golden or tiny or random or edge" > $OUT/pytest_parity.log 2>&1; echo "pytest rc=$?" >> $OUT/status
cat $OUT/variants.txt $OUT/status
