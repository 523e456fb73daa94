# round-2 GPU session d: new gate_bwd + epilogue TMEM batching: parity, launch list, bench
mkdir -p gpurun_out/r2e
make -s -j8 all 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 900 > gpurun_out/r2e/pytest.txt 2>&1; tail -3 gpurun_out/r2e/pytest.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2e/launches_tf.csv python tools/profile_step.py --config transformer --steps 2 > gpurun_out/r2e/ncu_tf.log 2>&1
python tools/launches.py gpurun_out/r2e/launches_tf.csv k_transpose > gpurun_out/r2e/launches_tf.txt; cat gpurun_out/r2e/launches_tf.txt
python bench.py > gpurun_out/r2e/bench_tf.json 2> gpurun_out/r2e/bench_tf.err; tail -c 1200 gpurun_out/r2e/bench_tf.json
