mkdir -p gpurun_out/r2p
make -s -j8 all 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_ffn.py -m gpu -q -x --timeout 300 > gpurun_out/r2p/pytest_ffn.txt 2>&1; tail -15 gpurun_out/r2p/pytest_ffn.txt
timeout 900 python bench.py --config grid3d --steps 10 --no-cpu-baseline > gpurun_out/r2p/bench_grid3d.json 2> gpurun_out/r2p/bench_grid3d.err; tail -c 900 gpurun_out/r2p/bench_grid3d.json; tail -3 gpurun_out/r2p/bench_grid3d.err
