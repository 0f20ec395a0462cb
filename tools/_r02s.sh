#!/bin/bash
OUT=gpurun_out/r02s; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for c in "c5 --coi=100" "c3 --coi=0,50,99" "c2"; do
  set -- $c
  timeout 900 python tools/perf_variants.py build_variants/lib_{cur,u2,u8,ppt6,walk8,tb40}.so --config=$1 $2 --reps=3 >> $OUT/variants.txt 2>&1
done
echo done > $OUT/status
