# round-2 GPU session j: early accumulator release; tests, launch list, bench
mkdir -p gpurun_out/r2j
make -s -j8 all 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_sgd.py tests/test_gpu_parity.py -m gpu -q -x --timeout 900 > gpurun_out/r2j/pytest.txt 2>&1; tail -4 gpurun_out/r2j/pytest.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2j/launches_tf.csv python tools/profile_step.py --config transformer --steps 2 > gpurun_out/r2j/ncu_tf.log 2>&1
python tools/launches.py gpurun_out/r2j/launches_tf.csv k_transpose > gpurun_out/r2j/launches_tf.txt; cat gpurun_out/r2j/launches_tf.txt
python bench.py > gpurun_out/r2j/bench_tf.json 2> gpurun_out/r2j/bench_tf.err; tail -c 1400 gpurun_out/r2j/bench_tf.json
