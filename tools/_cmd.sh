mkdir -p gpurun_out/r01at
python tools/perf_variants.py build_variants/lib_*.so --config=c4 --coi=0,40,79 --reps=2 > gpurun_out/r01at/variants_c4.txt 2>&1
cat gpurun_out/r01at/variants_*.txt
