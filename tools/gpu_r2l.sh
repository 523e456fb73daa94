mkdir -p gpurun_out/r2l
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
python tools/tc_wait.py transformer M=16 T=4096 2>&1 | tail -40
DBG=1 python tools/tc_wait.py transformer M=16 T=4096 2>&1 | grep -A4 "SEGK=1, EPI=4"
DMOE_NO_COLSUM_FUSE=1 python tools/tc_wait.py transformer M=16 T=4096 2>&1 | grep -A4 "SEGK=1, EPI=4"
make -s clean && make -s -j8 all 2>&1 | tail -2
