#!/bin/bash
# MODE_SEGPF (next span first table column prefetched during the span math) vs MODE_SEGMENT:
# c4 (3 COIs, all 80), then the GPU parity subset on the new default
OUT=gpurun_out/r02zr; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for c in "c4 --coi=0,40,79"; do
  set -- $c
  timeout 600 python tools/perf_variants.py build_variants/lib_pf0.so build_variants/lib_pf1.so build_variants/lib_pf0.so build_variants/lib_pf1.so --config=$1 $2 --reps=3 >> $OUT/variants.txt 2>&1
done
timeout 600 python tools/perf_variants.py build_variants/lib_pf0.so build_variants/lib_pf1.so --config=c4 --reps=2 >> $OUT/variants.txt 2>&1
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "golden or tiny or random or edge or table" > $OUT/pytest_parity.log 2>&1; echo "pytest rc=$?" >> $OUT/status
cat $OUT/variants.txt $OUT/status
