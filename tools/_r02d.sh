#!/bin/bash
OUT=gpurun_out/r02d; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 900 python tools/perf_variants.py build_variants/lib_{base,minb4,minb4t24,ppt2m4,ppt2m6,ppt8m2}.so --config=c5 --coi=100 --reps=2 > $OUT/variants_c5.txt 2>&1
timeout 600 python tools/perf_variants.py build_variants/lib_{base,minb4,minb4t24,ppt2m4,ppt2m6,ppt8m2}.so --config=c2 --reps=3 > $OUT/variants_c2.txt 2>&1
echo done > $OUT/status
