#!/bin/bash
OUT=gpurun_out/r02u; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "chain_groups or planned_work" > $OUT/pytest_new.txt 2>&1
timeout 2400 python tests/tools/kernel_mutants.py run > $OUT/kernel_mutants.jsonl 2>&1
echo done > $OUT/status
