mkdir -p gpurun_out/r01q
python -m pytest tests -m gpu -x -q > gpurun_out/r01q/pytest.log 2>&1; tail -2 gpurun_out/r01q/pytest.log
python tools/run_configs.py --configs c2,c4 > gpurun_out/r01q/configs.jsonl 2>&1; cat gpurun_out/r01q/configs.jsonl
