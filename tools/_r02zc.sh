#!/bin/bash
# final certification of the round-2 kernel (table sincospi): GPU suite, smoke, all configs, bench,
# launch list, ncu --set full of c4 (COI 40) and c5 (COI 100), all 17 kernel mutants
OUT=gpurun_out/r02zc; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status
timeout 900 python tools/run_configs.py > $OUT/all_configs.jsonl 2>&1; echo "configs rc=$?" >> $OUT/status
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dedup --no-extra > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?" >> $OUT/status
timeout 300 python tools/ncu_target.py --config c4 --coi 40 --reps 2 > $OUT/plain_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:integrand_kernel -s 3 -c 1 -o $OUT/prof_c4 python tools/ncu_target.py --config c4 --coi 40 --reps 2 > $OUT/ncu_c4.log 2>&1; echo "ncu c4 rc=$?" >> $OUT/status
timeout 300 python tools/ncu_target.py --config c5 --coi 100 --reps 2 > $OUT/plain_c5.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:integrand_kernel -s 3 -c 1 -o $OUT/prof_c5 python tools/ncu_target.py --config c5 --coi 100 --reps 2 > $OUT/ncu_c5.log 2>&1; echo "ncu c5 rc=$?" >> $OUT/status
timeout 1800 python tests/tools/kernel_mutants.py run > $OUT/mutants.jsonl 2>&1; echo "mutants rc=$?" >> $OUT/status
