#!/bin/bash
# (lib_step1 was built from a since-reverted tree with precomputed walk steps; see profiles/r02zf_*)
# precomputed envelope walk steps e^{-zeta_k g} (step1) vs computed in the table build (step0)
OUT=gpurun_out/r02zf; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for c in "c4 --coi=0,40,79" "c5 --coi=100" "c2" "c3 --coi=0,50,99"; do
  set -- $c
  timeout 600 python tools/perf_variants.py build_variants/lib_step0.so build_variants/lib_step1.so build_variants/lib_step0.so build_variants/lib_step1.so --config=$1 $2 --reps=3 >> $OUT/variants.txt 2>&1
done
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "golden or tiny or random or edge or c4 or precompute" > $OUT/pytest_parity.log 2>&1; echo "pytest rc=$?" >> $OUT/status
