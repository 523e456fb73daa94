# round-2 GPU session h: SGD tests, beam kernel profile, stress bench (chunked SGD, tied pool)
mkdir -p gpurun_out/r2h
make -s -j8 all 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_sgd.py -m gpu -q -x --timeout 900 > gpurun_out/r2h/pytest.txt 2>&1; tail -3 gpurun_out/r2h/pytest.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_beam_topk -c 1 -o gpurun_out/r2h/beam python tools/bench_routing.py --config transformer --n 1 > gpurun_out/r2h/ncu_beam.log 2>&1; tail -2 gpurun_out/r2h/ncu_beam.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tc_gemm -c 1 -o gpurun_out/r2h/gatetopk python tools/bench_routing.py --config transformer --n 1 > gpurun_out/r2h/ncu_gt.log 2>&1; tail -2 gpurun_out/r2h/ncu_gt.log
timeout 1200 python bench.py --config stress --steps 3 --warmup 3 > gpurun_out/r2h/bench_stress.json 2> gpurun_out/r2h/bench_stress.err; tail -c 2500 gpurun_out/r2h/bench_stress.json; tail -5 gpurun_out/r2h/bench_stress.err
