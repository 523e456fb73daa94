for nt in 64 128; do
  DMOE_TC_NT=$nt python tools/profile_step.py > /dev/null 2>&1 && DMOE_TC_NT=$nt ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_tc --log-file gpurun_out/nt$nt.csv python tools/profile_step.py > /dev/null 2>&1
  DMOE_TC_NT=$nt python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_nt$nt.json 2>/dev/null
done
