# final single-GPU session: full GPU test suite, smoke, then the round-2 evidence script
mkdir -p gpurun_out/final
make -s -j8 all 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/final/pytest_gpu.txt 2>&1; tail -2 gpurun_out/final/pytest_gpu.txt
timeout 600 python __graft_entry__.py smoke > gpurun_out/final/smoke.txt 2>&1; tail -1 gpurun_out/final/smoke.txt
bash tools/evidence_r2.sh
