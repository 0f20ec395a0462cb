#!/bin/bash
# fp32 variant (row a8): FADD2 with a negated operand for "- b_{k+2}" (ISRS_F32_ADD2=1) vs FFMA2 by -1
OUT=gpurun_out/r02zd; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for c in "c2" "c5 --coi=100" "c4 --coi=0,40,79" "c3 --coi=0,50,99"; do
  set -- $c
  timeout 600 python tools/perf_variants.py build_variants/lib_add0.so build_variants/lib_add2.so build_variants/lib_add0.so build_variants/lib_add2.so --config=$1 $2 --reps=3 --precision=32 >> $OUT/variants.txt 2>&1
done
ISRS_EGN_LIB=build_variants/lib_add2.so timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "fp32" > $OUT/pytest_fp32.log 2>&1; echo "pytest rc=$?" >> $OUT/status
