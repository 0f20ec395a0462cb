#!/bin/bash
# One gpurun session: GPU tests, smoke, bench, ncu launch list, one ncu --set full capture of the
# D-only integrand kernel.  Usage (from this container):
#   gpurun --timeout 1800 -- 'bash tools/gpu_run.sh [tag] [stages]'
# stages: any of t (pytest -m gpu) s (smoke) b (bench) l (ncu launch list) f (ncu full); default tsblf
set -u
TAG=${1:-run}
STAGES=${2:-tsblf}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"; lscpu | head -20 >> "$OUT/nproc.txt"
python -m paper_2412_11614_b200.build > "$OUT/build.log" 2>&1
if [[ $STAGES == *p* ]]; then
  for b in tools/dmma_probe tools/fp64_pipes; do [ -x $b ] && timeout 120 ./$b > "$OUT/$(basename $b).txt" 2>&1; done
  echo "probes rc=$?" >> "$OUT/status"
fi
if [[ $STAGES == *t* ]]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/status"
fi
if [[ $STAGES == *s* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/status"
fi
if [[ $STAGES == *b* ]]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/status"
fi
if [[ $STAGES == *l* ]]; then
  CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu ${BENCH_ARGS:-}"
  timeout 300 $CMD > "$OUT/plain_launch.log" 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file "$OUT/launches.csv" $CMD > "$OUT/ncu_launch.log" 2>&1
  echo "launches rc=$?" >> "$OUT/status"
fi
if [[ $STAGES == *f* ]]; then
  CMD="python tools/ncu_target.py ${NCU_CFG:---config c5 --coi 100} --reps 2"
  timeout 300 $CMD > "$OUT/plain_full.log" 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:integrand_kernel -s 3 -c 1 \
      -o "$OUT/prof" $CMD > "$OUT/ncu_full.log" 2>&1
  echo "ncu_full rc=$?" >> "$OUT/status"
fi
cat "$OUT/status"
