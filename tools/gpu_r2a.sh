set -x
mkdir -p gpurun_out/r2a
make -s -j8 all 2>&1 | tail -3
python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/r2a/pytest.txt 2>&1; tail -3 gpurun_out/r2a/pytest.txt
python bench.py > gpurun_out/r2a/bench_tf.json 2> gpurun_out/r2a/bench_tf.err; tail -c 3000 gpurun_out/r2a/bench_tf.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc_gemm<256, 1" -c 1 -o gpurun_out/r2a/segk_tfslice python tools/profile_step.py --config transformer --steps 1 --set M=16 T=4096 > gpurun_out/r2a/ncu_segk.log 2>&1; tail -3 gpurun_out/r2a/ncu_segk.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc_gemm<256, 0, 0, 1" -c 1 -o gpurun_out/r2a/fwd1_tfslice python tools/profile_step.py --config transformer --steps 1 --set M=16 T=4096 > gpurun_out/r2a/ncu_fwd.log 2>&1; tail -3 gpurun_out/r2a/ncu_fwd.log
