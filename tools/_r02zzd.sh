#!/bin/bash
# the split's SCI part at full size against the oracle's own-island value (c2, c3, c4, c5)
OUT=gpurun_out/r02zzd; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -s -p no:cacheprovider -k "sci_part_full_size" > $OUT/pytest_sci.log 2>&1; echo "pytest rc=$?" >> $OUT/status
