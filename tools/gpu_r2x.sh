# weight-gradient GEMM role waits at 64 / 256 / 1024 rows per expert (EXPERIMENTS build)
mkdir -p gpurun_out/r2x
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
python tools/tc_wait.py transformer M=16 T=4096 > gpurun_out/r2x/wait_k64.txt 2>&1
python tools/tc_wait.py transformer M=32 > gpurun_out/r2x/wait_k256.txt 2>&1
python tools/tc_wait.py transformer M=16 > gpurun_out/r2x/wait_k1024.txt 2>&1
grep -A4 "SEGK=1" gpurun_out/r2x/wait_k*.txt
make -s clean && make -s -j8 all 2>&1 | tail -2
