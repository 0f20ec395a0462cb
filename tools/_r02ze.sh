#!/bin/bash
# (lib_pf32 / lib_pf48 were built from a patched copy of csrc/ with MODE_SEGPF, reverted; see profiles/r02ze_*)
# c4: double-buffered prebuilt table (MODE_SEGPF) at 32 KB (20 rows per buffer) and 48 KB (30 rows per
# buffer) table budgets, each against the single-buffer kernel of the same build (ISRS_EGN_NO_SEGPF=1)
OUT=gpurun_out/r02ze; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for i in 1 2; do
  for lib in pf32 pf48; do
    ISRS_EGN_NO_SEGPF=1 timeout 300 python tools/perf_variants.py build_variants/lib_$lib.so --config=c4 --coi=0,40,79 --reps=3 | sed 's/^/nopf /' >> $OUT/variants.txt 2>&1
    timeout 300 python tools/perf_variants.py build_variants/lib_$lib.so --config=c4 --coi=0,40,79 --reps=3 | sed 's/^/pf /' >> $OUT/variants.txt 2>&1
  done
done
