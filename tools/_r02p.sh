#!/bin/bash
OUT=gpurun_out/r02p; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "tiny or edge or random_links or golden or chaining or c1 or streams or graph or shards or determinism or modes_parity or gn_reduction" > $OUT/pytest.txt 2>&1
timeout 900 python tools/perf_variants.py build_variants/lib_{grp4,mc}.so --config=c4 --coi=0,40,79 --reps=3 >> $OUT/variants.txt 2>&1
timeout 900 python tools/perf_variants.py build_variants/lib_{grp4,mc}.so --config=c2 --reps=3 >> $OUT/variants.txt 2>&1
echo done > $OUT/status
