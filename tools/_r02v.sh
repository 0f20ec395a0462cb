#!/bin/bash
OUT=gpurun_out/r02v; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
ISRS_EGN_LIB=build_variants/lib_chk.so timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/checked_pytest_gpu.txt 2>&1; echo "checked pytest rc=$?" >> $OUT/status
ISRS_EGN_LIB=build_variants/lib_chk.so timeout 600 python tools/sanitize_run.py > $OUT/checked_sanitize_run.txt 2>&1; echo "checked sanitize_run rc=$?" >> $OUT/status
timeout 300 compute-sanitizer --tool memcheck python tools/sanitize_run.py > $OUT/memcheck.txt 2>&1; echo "memcheck rc=$?" >> $OUT/status
