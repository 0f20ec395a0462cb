mkdir -p gpurun_out/r01aa
for spec in "c1:" "c3:50" "c5:100"; do
  cfg=${spec%%:*}; coi=${spec#*:}
  if [ -n "$coi" ]; then CMD="python tools/ncu_target.py --config $cfg --coi $coi --reps 2"; else CMD="python tools/ncu_target.py --config $cfg --reps 2"; fi
  timeout 300 $CMD > gpurun_out/r01aa/plain_$cfg.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:integrand_kernel -s 3 -c 1 -o gpurun_out/r01aa/prof_$cfg $CMD > gpurun_out/r01aa/ncu_$cfg.log 2>&1
  echo "$cfg rc=$?"
done
timeout 900 python tools/oracle_timing.py --configs c1 --sample c2,c3,c4,c5 --seconds 20 > gpurun_out/r01aa/oracle_timing.jsonl 2>&1
cat gpurun_out/r01aa/oracle_timing.jsonl | cut -c1-200
