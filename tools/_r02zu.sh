#!/bin/bash
# pinned staging of work-list uploads behind in-flight work: the async probe again, the stream /
# graph / COI-set-change tests, and the e2e leg (idle stream: pageable path, must not regress)
OUT=gpurun_out/r02zu; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for c in c3 c5; do timeout 600 python tools/async_probe.py --config $c >> $OUT/async_probe.jsonl 2>> $OUT/async_probe.err; echo "probe $c rc=$?" >> $OUT/status; done
timeout 900 python -m pytest tests -m gpu -x -q -s -k "coi_set or streams or graph or capture or shards or planned_work or tiny or c1" > $OUT/pytest_subset.log 2>&1; echo "pytest subset rc=$?" >> $OUT/status
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-dedup > $OUT/bench_short.json 2> $OUT/bench_short.err; echo "bench rc=$?" >> $OUT/status
