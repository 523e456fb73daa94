# per-phase time of the peer-memory expert-parallel step at 4 GPUs (transformer)
mkdir -p gpurun_out/ep4b
make -s -j8 all 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/ep_phases.py transformer > gpurun_out/ep4b/phases_transformer_ep4.txt 2>&1
tail -40 gpurun_out/ep4b/phases_transformer_ep4.txt
