bash tools/gpu_run.sh r01g t
python tools/dz_sweep.py --config c2 --dz 250,500,1000,2000,4000,7000 --ref 125 > gpurun_out/r01g/dz_sweep_c2.jsonl 2>&1
CMD="python tools/ncu_target.py --config c2 --reps 2 --precision 32"
timeout 300 $CMD > gpurun_out/r01g/plain_fp32.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:integrand_kernel -s 2 -c 1 -o gpurun_out/r01g/prof_fp32 $CMD > gpurun_out/r01g/ncu_fp32.log 2>&1
