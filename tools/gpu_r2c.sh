# round-2 GPU session c: thread-per-token beam + fused gate/top-k: parity, then bench
mkdir -p gpurun_out/r2c
make -s -j8 all 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -s --timeout 900 -x > gpurun_out/r2c/pytest.txt 2>&1; tail -5 gpurun_out/r2c/pytest.txt
grep -E "routing bit-exact|forced ReLU|FAIL|Error" gpurun_out/r2c/pytest.txt | head
python bench.py > gpurun_out/r2c/bench_tf.json 2> gpurun_out/r2c/bench_tf.err; tail -c 1500 gpurun_out/r2c/bench_tf.json; tail -3 gpurun_out/r2c/bench_tf.err
python bench.py --config mnist --steps 200 --no-cpu-baseline > gpurun_out/r2c/bench_mnist.json 2>&1; tail -c 800 gpurun_out/r2c/bench_mnist.json
