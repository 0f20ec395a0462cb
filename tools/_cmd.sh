mkdir -p gpurun_out/r01ap
python -m pytest tests -m gpu -x -q > gpurun_out/r01ap/pytest.log 2>&1; tail -1 gpurun_out/r01ap/pytest.log; grep -E "^E " gpurun_out/r01ap/pytest.log | head -3
python tools/perf_variants.py build_variants/lib_*.so --config=c4 --coi=0,40,79 --reps=2 > gpurun_out/r01ap/variants_c4.txt 2>&1
python tools/perf_variants.py build_variants/lib_*.so --config=c2 --reps=5 > gpurun_out/r01ap/variants_c2.txt 2>&1
cat gpurun_out/r01ap/variants_*.txt
