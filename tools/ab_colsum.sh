for v in 0 1; do
  if [ $v = 1 ]; then export DMOE_NO_COLSUM_FUSE=1; else unset DMOE_NO_COLSUM_FUSE; fi
  python tools/profile_step.py --config transformer --steps 2 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_tc|colsum" --log-file gpurun_out/ab_cs$v.csv python tools/profile_step.py --config transformer --steps 2 > /dev/null 2>&1
  python bench.py --config transformer --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_cs$v.json 2>&1
done
