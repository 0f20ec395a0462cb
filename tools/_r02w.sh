#!/bin/bash
OUT=gpurun_out/r02w; mkdir -p $OUT
timeout 900 python tools/perf_variants.py build_variants/lib_{cur2,norebuild}.so --config=c4 --coi=0,40,79 --reps=3 >> $OUT/variants.txt 2>&1
echo done > $OUT/status
