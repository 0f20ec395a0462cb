bash tools/gpu_run.sh r01ae f
python tools/dz_sweep.py --config c2 --dz 500,1000,2000,4000 --ref 250 > gpurun_out/r01ae/dz_sweep_c2.jsonl 2>&1
ISRS_EGN_LIB=build_variants/lib_prof.so python tools/ncu_target.py --config c2 --reps 2 > gpurun_out/r01ae/prof_c2.txt 2>&1
grep ISRS_PROF gpurun_out/r01ae/prof_c2.txt | sort -u
cut -c1-220 gpurun_out/r01ae/dz_sweep_c2.jsonl
