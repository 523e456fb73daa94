# round-2 GPU session b: new parity tests + ncu full captures of the transformer-shaped GEMMs
mkdir -p gpurun_out/r2b
make -s -j8 all 2>&1 | tail -3
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -s --timeout 900 -x > gpurun_out/r2b/pytest.txt 2>&1; tail -5 gpurun_out/r2b/pytest.txt
grep -E "routing bit-exact|forced ReLU" gpurun_out/r2b/pytest.txt
for sk in 1 4; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tc_gemm --launch-skip $sk -c 1 -o gpurun_out/r2b/tc_skip$sk python tools/profile_step.py --config transformer --steps 1 --set M=16 T=4096 > gpurun_out/r2b/ncu_$sk.log 2>&1; tail -2 gpurun_out/r2b/ncu_$sk.log
done
