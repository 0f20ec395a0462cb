#!/bin/bash
OUT=gpurun_out/r02aa; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 300 python tools/ncu_target.py --config c3 --coi 0,50,99 --reps 2 > $OUT/plain_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:integrand_kernel -s 3 -c 1 -o $OUT/prof_c3 python tools/ncu_target.py --config c3 --coi 0,50,99 --reps 2 > $OUT/ncu_c3.log 2>&1
echo "ncu rc=$?" > $OUT/status
