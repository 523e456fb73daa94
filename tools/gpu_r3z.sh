# smoke + ncu full of the beam search and the dispatch kernels at transformer
mkdir -p gpurun_out/r3z
make -s -j8 all 2>&1 | tail -2
timeout 600 python __graft_entry__.py smoke > gpurun_out/r3z/smoke.txt 2>&1; tail -1 gpurun_out/r3z/smoke.txt
ncu --set full --import-source on --clock-control none -k regex:"k_beam_topk|k_scan_chunks|k_rank|k_weights_hist" -s 4 -c 4 -o gpurun_out/r3z/beam_dispatch python tools/profile_step.py --config transformer --steps 2 > gpurun_out/r3z/ncu.log 2>&1; tail -1 gpurun_out/r3z/ncu.log
