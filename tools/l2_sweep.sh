for f in 0 32; do
  DMOE_TC_DEBUG=$f python tools/profile_step.py > /dev/null 2>&1 && DMOE_TC_DEBUG=$f ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_tc --log-file gpurun_out/l2_$f.csv python tools/profile_step.py > /dev/null 2>&1
  DMOE_TC_DEBUG=$f python tools/profile_step.py --config transformer --steps 2 > /dev/null 2>&1 && DMOE_TC_DEBUG=$f ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_tc --log-file gpurun_out/l2tf_$f.csv python tools/profile_step.py --config transformer --steps 2 > /dev/null 2>&1
done
python -m pytest tests/test_gpu_ffn.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
