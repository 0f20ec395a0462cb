#!/bin/bash
# HEAD (fp32 FADD2) GPU suite; the -DISRS_CHECK bounds-checked build on the whole GPU suite and every
# mode; ncu --set full of the fp32 variant (row a8) on c5 COI 100 and on c2
OUT=gpurun_out/r02zg; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status
ISRS_EGN_LIB=build_variants/lib_chk.so timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/checked_pytest_gpu.txt 2>&1; echo "checked pytest rc=$?" >> $OUT/status
ISRS_EGN_LIB=build_variants/lib_chk.so timeout 600 python tools/sanitize_run.py > $OUT/checked_sanitize_run.txt 2>&1; echo "checked sanitize_run rc=$?" >> $OUT/status
timeout 300 python tools/ncu_target.py --config c5 --coi 100 --reps 2 --precision 32 > $OUT/plain_c5_fp32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:integrand_kernel -s 3 -c 1 -o $OUT/prof_c5_fp32 python tools/ncu_target.py --config c5 --coi 100 --reps 2 --precision 32 > $OUT/ncu_c5_fp32.log 2>&1; echo "ncu c5 fp32 rc=$?" >> $OUT/status
timeout 600 ncu --set full --clock-control none --import-source on -k regex:integrand_kernel -s 3 -c 1 -o $OUT/prof_c2_fp32 python tools/ncu_target.py --config c2 --reps 2 --precision 32 > $OUT/ncu_c2_fp32.log 2>&1; echo "ncu c2 fp32 rc=$?" >> $OUT/status
