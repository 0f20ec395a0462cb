#!/bin/bash
# does nli return to the host before the GPU finishes when the COI set changes? (tools/async_probe.py)
OUT=gpurun_out/r02zt; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for c in c3 c5; do timeout 600 python tools/async_probe.py --config $c >> $OUT/async_probe.jsonl 2>> $OUT/async_probe.err; echo "probe $c rc=$?" >> $OUT/status; done
