#!/bin/bash
# the -DISRS_CHECK build (device bounds checks on every shared-memory index family, trap on violation)
# on the split tests, the async / stream tests and the fast parity subset
OUT=gpurun_out/r02zz; mkdir -p $OUT
ISRS_EGN_LIB=$PWD/build_variants/lib_check.so timeout 1200 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "split or coi_set or streams or graph or tiny or edge or random_links or c1_full or planned_work or chain_groups or problem" > $OUT/checked_pytest.log 2>&1; echo "checked pytest rc=$?" >> $OUT/status
ISRS_EGN_LIB=$PWD/build_variants/lib_check.so timeout 600 python tools/sanitize_run.py > $OUT/checked_sanitize_run.log 2>&1; echo "checked sanitize_run rc=$?" >> $OUT/status
