# role waits after the epilogue changes: transformer slice and full transformer (EXPERIMENTS build)
mkdir -p gpurun_out/r3b
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
python tools/tc_wait.py transformer M=16 T=4096 > gpurun_out/r3b/wait_k64.txt 2>&1
python tools/tc_wait.py transformer > gpurun_out/r3b/wait_full.txt 2>&1
grep -A5 "SEGK=1, EPI=4" gpurun_out/r3b/wait_*.txt
make -s clean && make -s -j8 all 2>&1 | tail -2
