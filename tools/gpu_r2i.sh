# round-2 GPU session i: beam lists+merge, 16-warp weight-gradient epilogue: tests, timing, profiles
mkdir -p gpurun_out/r2i
make -s -j8 all 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_routing.py tests/test_gpu_ffn.py tests/test_gpu_sgd.py tests/test_gpu_parity.py -m gpu -q -x --timeout 900 > gpurun_out/r2i/pytest.txt 2>&1; tail -4 gpurun_out/r2i/pytest.txt
python tools/bench_routing.py --config transformer 2>&1 | tail -4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_beam_topk -c 1 -o gpurun_out/r2i/beam python tools/bench_routing.py --config transformer --n 1 > gpurun_out/r2i/ncu_beam.log 2>&1; tail -1 gpurun_out/r2i/ncu_beam.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2i/launches_tf.csv python tools/profile_step.py --config transformer --steps 2 > gpurun_out/r2i/ncu_tf.log 2>&1
python tools/launches.py gpurun_out/r2i/launches_tf.csv k_transpose > gpurun_out/r2i/launches_tf.txt; cat gpurun_out/r2i/launches_tf.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tc_gemm --launch-skip 4 -c 1 -o gpurun_out/r2i/segk_slice python tools/profile_step.py --config transformer --steps 1 --set M=16 T=4096 > gpurun_out/r2i/ncu_segk.log 2>&1; tail -1 gpurun_out/r2i/ncu_segk.log
