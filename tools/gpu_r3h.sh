# ncu full capture of the full-size transformer weight-gradient GEMM (product build)
mkdir -p gpurun_out/r3h
make -s -j8 all 2>&1 | tail -2
ncu --set full --import-source on --clock-control none -k regex:k_tc_gemm -s 11 -c 1 -o gpurun_out/r3h/segk_full python tools/profile_step.py --config transformer --steps 2 > gpurun_out/r3h/ncu.log 2>&1; tail -2 gpurun_out/r3h/ncu.log
