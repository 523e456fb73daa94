for f in 0 16; do
  DMOE_TC_DEBUG=$f python tools/profile_step.py > /dev/null 2>&1 && DMOE_TC_DEBUG=$f ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_tc --log-file gpurun_out/pf$f.csv python tools/profile_step.py > /dev/null 2>&1
done
python -m pytest tests/test_gpu_ffn.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/bench_pf.json 2>&1
