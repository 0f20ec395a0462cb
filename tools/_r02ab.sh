#!/bin/bash
OUT=gpurun_out/r02ab; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 1200 python tests/tools/golden_parity.py > $OUT/golden_parity.jsonl 2>&1; echo "golden rc=$?" >> $OUT/status
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -s -k "golden" > $OUT/pytest_golden.txt 2>&1; echo "pytest rc=$?" >> $OUT/status
