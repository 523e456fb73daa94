for bn in auto 128 256; do
  if [ $bn = auto ]; then unset DMOE_TC_BN; else export DMOE_TC_BN=$bn; fi
  python tools/profile_step.py > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_tc --log-file gpurun_out/bn$bn.csv python tools/profile_step.py > /dev/null 2>&1
done
unset DMOE_TC_BN
python -m pytest tests/test_gpu_ffn.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/bench_bn.json 2>&1
