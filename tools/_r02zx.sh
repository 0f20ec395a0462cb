#!/bin/bash
# the three SCI / XCI / MCI split kernel mutants against the fast GPU parity subset (each must fail it),
# and the unmutated HEAD on the same subset (must pass)
OUT=gpurun_out/r02zx; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 1500 python tests/tools/kernel_mutants.py run split_filter_k2 > $OUT/kernel_mutants_k2.jsonl 2> $OUT/kernel_mutants.err; echo "mutants rc=$?" >> $OUT/status
