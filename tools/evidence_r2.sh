#!/bin/bash
# Round-2 final evidence (one GPU): bench lines for every workload and the alive-mask sweep, ncu
# launch lists with DRAM bytes (cold cache, serialised: per-kernel share and traffic), the launch
# list of bench.py itself (the contract's command), one ncu --set full capture of the dominant
# kernel (the transformer weight-gradient GEMM).  Outputs under gpurun_out/ev2/.
mkdir -p gpurun_out/ev2
make -s -j8 all 2>&1 | tail -2
line() {
  python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$2', round(d['value']), round(d['ms_per_step'], 3), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'], 3), d['clocks'])"
}
for cfg in transformer mnist grid3d mnist_block transformer_block stress; do
  st=20; w=5
  [ $cfg = mnist ] && st=400
  [ $cfg = mnist_block ] && st=100
  [ $cfg = stress ] && st=3 && w=3
  [ $cfg = transformer_block ] && st=10
  python bench.py --config $cfg --steps $st --warmup $w > gpurun_out/ev2/bench_$cfg.json 2> gpurun_out/ev2/bench_$cfg.err
  line gpurun_out/ev2/bench_$cfg.json $cfg
done
for df in 0.1 0.3; do
  python bench.py --config transformer --dead-frac $df --steps 20 --no-cpu-baseline > gpurun_out/ev2/bench_transformer_dead$df.json 2> gpurun_out/ev2/bench_transformer_dead$df.err
  line gpurun_out/ev2/bench_transformer_dead$df.json dead$df
done
python bench.py --config transformer --fail-frac 0.3 --steps 20 --no-cpu-baseline > gpurun_out/ev2/bench_transformer_fail0.3.json 2> gpurun_out/ev2/bench_transformer_fail0.3.err
line gpurun_out/ev2/bench_transformer_fail0.3.json fail0.3
for cfg in transformer grid3d; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/ev2/launches_$cfg.csv python tools/profile_step.py --config $cfg --steps 2 > gpurun_out/ev2/ncu_$cfg.log 2>&1
  python tools/launches.py gpurun_out/ev2/launches_$cfg.csv > gpurun_out/ev2/launches_$cfg.txt
  python tools/traffic.py gpurun_out/ev2/launches_$cfg.csv $cfg gpurun_out/ev2/traffic_$cfg.json > gpurun_out/ev2/traffic_$cfg.txt
  tail -1 gpurun_out/ev2/launches_$cfg.txt
done
# the contract's launch list: the bench command itself (cold cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev2/ncu_bench_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ev2/ncu_bench.log 2>&1
tail -1 gpurun_out/ev2/ncu_bench.log
# dominant kernel: the transformer weight-gradient GEMM (k_tc_gemm<256, 1, 1, 4>), one full capture
ncu --set full --import-source on --clock-control none -k regex:k_tc_gemm -s 11 -c 1 -o gpurun_out/ev2/segk_transformer \
  python tools/profile_step.py --config transformer --steps 2 > gpurun_out/ev2/ncu_full.log 2>&1
tail -1 gpurun_out/ev2/ncu_full.log
echo evidence-done
