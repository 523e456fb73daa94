# round-2 GPU session f: routing tests, parity, launch list, bench
mkdir -p gpurun_out/r2f
make -s -j8 all 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_routing.py tests/test_gpu_parity.py tests/test_gpu_ffn.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 900 > gpurun_out/r2f/pytest.txt 2>&1; tail -15 gpurun_out/r2f/pytest.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2f/launches_tf.csv python tools/profile_step.py --config transformer --steps 2 > gpurun_out/r2f/ncu_tf.log 2>&1
python tools/launches.py gpurun_out/r2f/launches_tf.csv k_transpose > gpurun_out/r2f/launches_tf.txt; cat gpurun_out/r2f/launches_tf.txt
python bench.py > gpurun_out/r2f/bench_tf.json 2> gpurun_out/r2f/bench_tf.err; tail -c 1000 gpurun_out/r2f/bench_tf.json
