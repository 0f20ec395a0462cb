bash tools/gpu_run.sh r01f tb
python tools/perf_variants.py build_variants/lib_*.so --reps=3 > gpurun_out/r01f/variants_c2.txt 2>&1
python tools/perf_variants.py build_variants/lib_*.so --config=c5 --coi=100 --reps=1 > gpurun_out/r01f/variants_c5.txt 2>&1
python bench.py --precision 32 --no-cpu > gpurun_out/r01f/bench_fp32.json 2> gpurun_out/r01f/bench_fp32.err
