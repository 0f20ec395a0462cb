#!/bin/bash
OUT=gpurun_out/r02q; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 300 python tools/ncu_target.py --config c4 --coi 40 --reps 2 > $OUT/plain_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:integrand_kernel -s 3 -c 1 -o $OUT/prof_c4 python tools/ncu_target.py --config c4 --coi 40 --reps 2 > $OUT/ncu_c4.log 2>&1
echo "ncu rc=$?" > $OUT/status
