#!/bin/bash
# (ran a MODE_SEGPF build that is not in the tree: the experiment was reverted, see profiles/r02zb_*)
# MODE_SEGPF (double-buffered prebuilt table on multi-class links) vs the single-buffer kernel
OUT=gpurun_out/r02zb; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for i in 1 2; do
  ISRS_EGN_NO_SEGPF=1 timeout 300 python tools/perf_variants.py build_variants/lib_pf1.so --config=c4 --coi=0,40,79 --reps=3 | sed 's/^/nopf /' >> $OUT/variants.txt 2>&1
  timeout 300 python tools/perf_variants.py build_variants/lib_pf1.so --config=c4 --coi=0,40,79 --reps=3 | sed 's/^/pf /' >> $OUT/variants.txt 2>&1
done
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "golden or tiny or random or edge or shards or mirror or c4" > $OUT/pytest_parity.log 2>&1; echo "pytest rc=$?" >> $OUT/status
timeout 1500 python tests/tools/kernel_mutants.py run cistab_index cistab_sin_sign cistab_cos_term > $OUT/mutants.jsonl 2>&1; echo "mutants rc=$?" >> $OUT/status
