mkdir -p gpurun_out/r2n
make -s -j8 all 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_ffn3.py -m gpu -q -x -s --timeout 900 > gpurun_out/r2n/pytest.txt 2>&1; tail -30 gpurun_out/r2n/pytest.txt
