#!/bin/bash
OUT=gpurun_out/r02t; mkdir -p $OUT
timeout 900 python tools/perf_variants.py build_variants/lib_{cur,minb4,minb4t24,ppt2m4,ppt2m6,ppt8m2}.so --config=c4 --coi=0,40,79 --reps=3 >> $OUT/variants.txt 2>&1
echo done > $OUT/status
