#!/bin/bash
# all 22 kernel mutants (19 earlier + 3 of the SCI / XCI / MCI split), rebuilt from HEAD, against the fast
# GPU parity subset (each must fail it); HEAD itself passed the same subset in r02zx
OUT=gpurun_out/r02zzb; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 2400 python tests/tools/kernel_mutants.py run > $OUT/kernel_mutants.jsonl 2> $OUT/kernel_mutants.err; echo "mutants rc=$?" >> $OUT/status
ISRS_EGN_LIB=$PWD/build_variants/lib_check.so timeout 600 python tools/sanitize_run.py > $OUT/checked_sanitize_run.log 2>&1; echo "checked sanitize_run rc=$?" >> $OUT/status
