# role waits of the full-size transformer dW GEMM with the current code (EXPERIMENTS build)
mkdir -p gpurun_out/r3t
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
python tools/tc_wait.py transformer > gpurun_out/r3t/wait_full.txt 2>&1
grep -A6 "SEGK=1, EPI=4" gpurun_out/r3t/wait_full.txt
make -s clean && make -s -j8 all 2>&1 | tail -2
