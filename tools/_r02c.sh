#!/bin/bash
# r02c: phase timers on c5 (COI 100) and a dz sweep for the T(K) = a K + b split
OUT=gpurun_out/r02c; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
ISRS_EGN_LIB=build_variants/lib_prof.so timeout 300 python tools/ncu_target.py --config c5 --coi 100 --reps 2 > $OUT/prof_c5.txt 2>&1
ISRS_EGN_LIB=build_variants/lib_prof.so timeout 300 python tools/ncu_target.py --config c4 --coi 0,40,79 --reps 2 > $OUT/prof_c4.txt 2>&1
timeout 600 python tools/dz_sweep.py --config c5 --coi 100 --dz 500,800,1000,2000 --ref 500 --reps 2 > $OUT/dz_c5.jsonl 2>&1
echo done > $OUT/status
