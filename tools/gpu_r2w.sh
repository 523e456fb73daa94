# per-rank compute of EP4 / EP16-like shapes on one GPU: launch lists (256 and 1024 rows per expert)
mkdir -p gpurun_out/r2w
make -s -j8 all 2>&1 | tail -3
for m in 32 16; do
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 60 --csv --log-file gpurun_out/r2w/launches_m$m.csv python tools/profile_step.py --config transformer --steps 2 --set M=$m > gpurun_out/r2w/ncu_m$m.log 2>&1
python tools/launches.py gpurun_out/r2w/launches_m$m.csv > gpurun_out/r2w/launches_m$m.txt; cat gpurun_out/r2w/launches_m$m.txt
done
