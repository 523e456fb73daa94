mkdir -p gpurun_out/r2k
make -s -j8 all 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_routing.py tests/test_gpu_parity.py -m gpu -q -x --timeout 900 > gpurun_out/r2k/pytest.txt 2>&1; tail -3 gpurun_out/r2k/pytest.txt
python tools/bench_routing.py --config transformer 2>&1 | tail -4
python tools/bench_routing.py --config grid3d 2>&1 | tail -4
bash tools/segk_exp.sh
