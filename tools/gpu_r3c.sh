# CTA-0 timeline of the weight-gradient GEMM (transformer slice), EXPERIMENTS build
mkdir -p gpurun_out/r3c
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
KERNEL=256,1,4 NT=32 python tools/tc_probe.py transformer M=16 T=4096 > gpurun_out/r3c/probe_k64.txt 2>&1
cat gpurun_out/r3c/probe_k64.txt | tail -36
make -s clean && make -s -j8 all 2>&1 | tail -2
