#!/bin/bash
# One GPU session of round evidence: gpu tests, bench lines for the configs, ncu launch lists
# with DRAM bytes (cold cache, serialised: per-kernel share and traffic, not absolute step time),
# one ncu --set full capture of the step's tcgen05 GEMMs, the microbenchmarks, pipeline cycles.
mkdir -p gpurun_out/ev
python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/ev/pytest.txt 2>&1
tail -3 gpurun_out/ev/pytest.txt
for cfg in ${CFGS:-mnist transformer grid3d}; do
  st=400; [ $cfg != mnist ] && st=20
  python bench.py --config $cfg --steps $st > gpurun_out/ev/bench_$cfg.json 2> gpurun_out/ev/bench_$cfg.err
  python -c "
import json; d=json.loads(open('gpurun_out/ev/bench_$cfg.json').read().strip().splitlines()[-1])
print('$cfg', round(d['value']), d['ms_per_step'], 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'], 3), d['clocks'])"
done
for cfg in ${NCU_CFGS:-mnist transformer}; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/ev/launches_$cfg.csv python tools/profile_step.py --config $cfg --steps 2 > gpurun_out/ev/ncu_$cfg.log 2>&1
  python tools/launches.py gpurun_out/ev/launches_$cfg.csv > gpurun_out/ev/launches_$cfg.txt
  tail -1 gpurun_out/ev/launches_$cfg.txt
done
if [ -z "$SKIP_FULL" ]; then
  ncu --set full --import-source on --clock-control none -k regex:k_tc_gemm --launch-skip 7 -c 7 \
    -o gpurun_out/ev/gemms_mnist python tools/profile_step.py --config mnist --steps 2 > gpurun_out/ev/ncu_full.log 2>&1
  tail -1 gpurun_out/ev/ncu_full.log
fi
./tools/hbm_bw > gpurun_out/ev/hbm_bw.txt 2>&1
./tools/mma_rate > gpurun_out/ev/mma_rate.txt 2>&1
python tools/tc_wait.py mnist > gpurun_out/ev/wait_mnist.txt 2>&1
python tools/tc_wait.py transformer > gpurun_out/ev/wait_transformer.txt 2>&1
echo evidence-done
