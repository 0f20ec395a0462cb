#!/bin/bash
# NEXT-4a dedup: closed form in its own instantiation MODE_SEGDDL for runs > 32 spans (dd4) vs the loop (dd0)
OUT=gpurun_out/r02zl; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for i in 1 2; do for lib in dd0 dd4; do
  ISRS_EGN_LIB=build_variants/lib_$lib.so timeout 300 python tools/dedup_time.py --config c5 --coi 0,100,199 >> $OUT/dedup.jsonl 2>&1
  ISRS_EGN_LIB=build_variants/lib_$lib.so timeout 300 python tools/dedup_time.py --config c2 >> $OUT/dedup.jsonl 2>&1
  ISRS_EGN_LIB=build_variants/lib_$lib.so timeout 300 python tools/dedup_time.py --config c3 --coi 0,50,99 >> $OUT/dedup.jsonl 2>&1
done; done
for m in "" "--mirror"; do ISRS_EGN_LIB=build_variants/lib_dd4.so timeout 300 python tools/dedup_time.py --config c5 $m >> $OUT/dedup.jsonl 2>&1; done
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "dedup or mirror or random" > $OUT/pytest_dedup.log 2>&1; echo "pytest rc=$?" >> $OUT/status
