bash tools/gpu_run.sh r01j tsb
