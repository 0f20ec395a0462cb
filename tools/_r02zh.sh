#!/bin/bash
# run-to-run spread of the headline bench (3 fresh processes), the fp32 variant's bench line, and the
# reference arm (the oracle on the box's cores) on the final code
OUT=gpurun_out/r02zh; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for i in 1 2 3; do timeout 900 python bench.py --no-cpu > $OUT/bench_$i.json 2> $OUT/bench_$i.err; echo "bench $i rc=$?" >> $OUT/status; done
timeout 900 python bench.py --precision 32 --no-cpu > $OUT/bench_fp32.json 2> $OUT/bench_fp32.err; echo "bench32 rc=$?" >> $OUT/status
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?" >> $OUT/status
