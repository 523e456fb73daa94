# role waits of the weight-gradient GEMM pipeline skeleton (no loads / MMA / TMEM loads / stores)
mkdir -p gpurun_out/r3n
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
DMOE_TC_DEBUG_SEGK=519 python tools/tc_wait.py transformer M=16 T=4096 > gpurun_out/r3n/wait_skel_k64.txt 2>&1
DMOE_NO_COLSUM_FUSE=1 DMOE_TC_DEBUG_SEGK=519 python tools/tc_wait.py transformer M=16 T=4096 > gpurun_out/r3n/wait_skel_nocs_k64.txt 2>&1
DMOE_NO_COLSUM_FUSE=1 python tools/tc_wait.py transformer M=16 T=4096 > gpurun_out/r3n/wait_nocs_k64.txt 2>&1
grep -A6 "SEGK=1, EPI=4" gpurun_out/r3n/wait_*.txt
make -s clean && make -s -j8 all 2>&1 | tail -2
