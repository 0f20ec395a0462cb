#!/bin/bash
OUT=gpurun_out/r02k; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -s -k "full_size_region_parity" > $OUT/region_parity.txt 2>&1
timeout 900 python tests/tools/golden_parity.py > $OUT/golden_parity.jsonl 2>&1
echo done > $OUT/status
