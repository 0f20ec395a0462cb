mkdir -p gpurun_out/r01r
python -m pytest tests -m gpu -x -q > gpurun_out/r01r/pytest.log 2>&1; tail -2 gpurun_out/r01r/pytest.log
python tools/run_configs.py --configs c2,c4 > gpurun_out/r01r/configs.jsonl 2>&1; cut -c1-300 gpurun_out/r01r/configs.jsonl
