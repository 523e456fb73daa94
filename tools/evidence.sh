#!/bin/bash
# One GPU session of round evidence: gpu tests, bench lines for the configs, ncu launch lists
# with DRAM bytes (cold cache, serialised: per-kernel share and traffic, not absolute step time).
mkdir -p gpurun_out/ev
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev/pytest.txt
cat gpurun_out/ev/pytest.txt
for cfg in ${CFGS:-mnist transformer grid3d}; do
  st=400; [ $cfg != mnist ] && st=20
  python bench.py --config $cfg --steps $st > gpurun_out/ev/bench_$cfg.json 2> gpurun_out/ev/bench_$cfg.err
  tail -c 300 gpurun_out/ev/bench_$cfg.json; echo
done
for cfg in ${NCU_CFGS:-mnist transformer}; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/ev/launches_$cfg.csv python tools/profile_step.py --config $cfg --steps 2 > gpurun_out/ev/ncu_$cfg.log 2>&1
  python tools/launches.py gpurun_out/ev/launches_$cfg.csv > gpurun_out/ev/launches_$cfg.txt
  tail -3 gpurun_out/ev/launches_$cfg.txt
done
