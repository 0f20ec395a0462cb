#!/bin/bash
# NEXT-4a dedup: closed-form phased-array sum (dd1) vs the G-1 complex products (dd0)
OUT=gpurun_out/r02zi; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for i in 1 2; do for lib in dd0 dd1; do
  ISRS_EGN_LIB=build_variants/lib_$lib.so timeout 300 python tools/dedup_time.py --config c5 >> $OUT/dedup.jsonl 2>&1
  ISRS_EGN_LIB=build_variants/lib_$lib.so timeout 300 python tools/dedup_time.py --config c5 --mirror >> $OUT/dedup.jsonl 2>&1
  ISRS_EGN_LIB=build_variants/lib_$lib.so timeout 300 python tools/dedup_time.py --config c2 >> $OUT/dedup.jsonl 2>&1
done; done
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "dedup or mirror" > $OUT/pytest_dedup.log 2>&1; echo "pytest rc=$?" >> $OUT/status
