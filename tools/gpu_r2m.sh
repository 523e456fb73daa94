mkdir -p gpurun_out/r2m
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
KERNEL="256,1,4" NT=24 python tools/tc_probe.py transformer M=16 T=4096 2>&1 | tail -30
make -s clean && make -s -j8 all 2>&1 | tail -2
