#!/bin/bash
OUT=gpurun_out/r02e; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "tiny or edge or random_links or golden or chaining or c1 or streams or graph" > $OUT/pytest.txt 2>&1
timeout 900 python tools/perf_variants.py build_variants/lib_{base,grp,grpppt8}.so --config=c5 --coi=100 --reps=2 > $OUT/variants_c5.txt 2>&1
timeout 600 python tools/perf_variants.py build_variants/lib_{base,grp,grpppt8}.so --config=c2 --reps=3 > $OUT/variants_c2.txt 2>&1
timeout 600 python tools/perf_variants.py build_variants/lib_{base,grp,grpppt8}.so --config=c3 --coi=0,50,99 --reps=3 > $OUT/variants_c3.txt 2>&1
echo done > $OUT/status
