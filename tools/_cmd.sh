mkdir -p gpurun_out/r01ac
python tools/perf_variants.py build_variants/lib_*.so --reps=5 > gpurun_out/r01ac/variants_c2.txt 2>&1
python tools/perf_variants.py build_variants/lib_*.so --config=c5 --coi=100 --reps=1 > gpurun_out/r01ac/variants_c5.txt 2>&1
python tools/perf_variants.py build_variants/lib_*.so --config=c4 --coi=0,40,79 --reps=2 > gpurun_out/r01ac/variants_c4.txt 2>&1
cat gpurun_out/r01ac/variants_*.txt
