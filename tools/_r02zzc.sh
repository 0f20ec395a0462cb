#!/bin/bash
# SCI / XCI / MCI shares of every channel of c2, c3 and c5 (the 20 THz / 50-span link), with the unsplit eta as check
OUT=gpurun_out/r02zzc; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
for c in c2 c3 c5; do timeout 900 python tools/split_profile.py --config $c --check > $OUT/split_$c.json 2> $OUT/split_$c.err; echo "split $c rc=$?" >> $OUT/status; done
