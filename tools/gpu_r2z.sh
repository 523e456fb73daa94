# ncu full capture (source-level stall sampling) of the weight-gradient GEMM on a transformer-shaped slice
mkdir -p gpurun_out/r2z
make -s -j8 all 2>&1 | tail -2
ncu --set full --import-source on --clock-control none -k regex:k_tc_gemm -s 11 -c 1 -o gpurun_out/r2z/segk_k64 python tools/profile_step.py --config transformer --steps 2 --set M=16 T=4096 > gpurun_out/r2z/ncu.log 2>&1; tail -2 gpurun_out/r2z/ncu.log
