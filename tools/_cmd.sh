mkdir -p gpurun_out/r01af
python tools/perf_variants.py build_variants/lib_*.so --reps=5 > gpurun_out/r01af/variants_c2.txt 2>&1
python tools/perf_variants.py build_variants/lib_*.so --config=c5 --coi=100 --reps=1 > gpurun_out/r01af/variants_c5.txt 2>&1
cat gpurun_out/r01af/variants_*.txt
