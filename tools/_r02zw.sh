#!/bin/bash
# SCI / XCI / MCI split (ISRS_EGN_FLAG_SPLIT): its GPU parity tests, then the fast parity subset
OUT=gpurun_out/r02zw; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -s -k "split" > $OUT/pytest_split.log 2>&1; echo "pytest split rc=$?" >> $OUT/status
timeout 900 python -m pytest tests -m gpu -x -q -k "tiny or edge or random or c1 or streams or planned_work or coi_set or shards" > $OUT/pytest_subset.log 2>&1; echo "pytest subset rc=$?" >> $OUT/status
