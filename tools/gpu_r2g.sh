# round-2 GPU session g: gate_bwd smem-slice dx, SGD tests, routing timing, launch list, bench
mkdir -p gpurun_out/r2g
make -s -j8 all 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_sgd.py tests/test_gpu_parity.py tests/test_gpu_routing.py -m gpu -q -x --timeout 900 > gpurun_out/r2g/pytest.txt 2>&1; tail -15 gpurun_out/r2g/pytest.txt
python tools/bench_routing.py --config transformer 2>&1 | tail -4
python tools/bench_routing.py --config mnist 2>&1 | tail -4
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2g/launches_tf.csv python tools/profile_step.py --config transformer --steps 2 > gpurun_out/r2g/ncu_tf.log 2>&1
python tools/launches.py gpurun_out/r2g/launches_tf.csv k_transpose > gpurun_out/r2g/launches_tf.txt; cat gpurun_out/r2g/launches_tf.txt
