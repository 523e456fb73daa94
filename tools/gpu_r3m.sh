# role waits of the weight-gradient GEMM pipeline skeleton (no loads / MMA / TMEM loads / stores)
mkdir -p gpurun_out/r3m
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
DMOE_TC_DEBUG_SEGK=519 python tools/tc_wait.py transformer M=16 T=4096 > gpurun_out/r3m/wait_skel_k64.txt 2>&1
DMOE_TC_DEBUG_SEGK=519 KERNEL=256,1,4 NT=32 python tools/tc_probe.py transformer M=16 T=4096 > gpurun_out/r3m/probe_skel_k64.txt 2>&1
grep -A6 "SEGK=1, EPI=4" gpurun_out/r3m/wait_skel_k64.txt; tail -20 gpurun_out/r3m/probe_skel_k64.txt
make -s clean && make -s -j8 all 2>&1 | tail -2
