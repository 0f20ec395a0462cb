#!/bin/bash
# the 19 planted CUDA-source slips, rebuilt from HEAD's sources, against the GPU parity subset
OUT=gpurun_out/r02zn; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 2400 python tests/tools/kernel_mutants.py run > $OUT/mutants.jsonl 2>&1; echo "mutants rc=$?" >> $OUT/status
timeout 600 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "tiny or edge or random_links or c1_full or streams or planned_work or chain_groups or (golden and c2_eta) or dedup_closed_form" > $OUT/pytest_subset_head.log 2>&1; echo "head subset rc=$?" >> $OUT/status
