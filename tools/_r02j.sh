#!/bin/bash
OUT=gpurun_out/r02j; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "tiny or edge or random_links or golden or chaining or c1 or streams or graph or shards or determinism or gn_reduction or unit_link" > $OUT/pytest.txt 2>&1
for c in "c5 --coi=100" "c2" "c3 --coi=0,50,99" "c4 --coi=0,40,79"; do
  set -- $c
  timeout 900 python tools/perf_variants.py build_variants/lib_{grp4,shfl}.so --config=$1 $2 --reps=3 >> $OUT/variants.txt 2>&1
done
echo done > $OUT/status
