# weight-gradient GEMM role waits incl. epilogue phases and fix-up warp (EXPERIMENTS build)
mkdir -p gpurun_out/r2y
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
python tools/tc_wait.py transformer M=16 T=4096 > gpurun_out/r2y/wait_k64.txt 2>&1
python tools/tc_wait.py transformer M=32 > gpurun_out/r2y/wait_k256.txt 2>&1
python tools/tc_wait.py transformer M=16 > gpurun_out/r2y/wait_k1024.txt 2>&1
DMOE_NO_COLSUM_FUSE=1 python tools/tc_wait.py transformer M=16 > gpurun_out/r2y/wait_k1024_nocs.txt 2>&1
DMOE_NO_COLSUM_FUSE=1 python tools/tc_wait.py transformer M=32 > gpurun_out/r2y/wait_k256_nocs.txt 2>&1
grep -A5 "SEGK=1, EPI=4" gpurun_out/r2y/wait_k*.txt
make -s clean && make -s -j8 all 2>&1 | tail -2
