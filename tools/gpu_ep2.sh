# 2-GPU session: expert-parallel parity (NCCL + NVLink peer exchange) and EP bench lines
mkdir -p gpurun_out/ep2
make -s -j8 all 2>&1 | tail -3
nvidia-smi topo -m > gpurun_out/ep2/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ep.py -m gpu -v --timeout 600 > gpurun_out/ep2/pytest_ep.txt 2>&1; tail -8 gpurun_out/ep2/pytest_ep.txt
for cfg in transformer mnist; do
  st=20; [ $cfg = mnist ] && st=200
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --config $cfg --steps $st --warmup 5 > gpurun_out/ep2/bench_${cfg}_ep2.json 2> gpurun_out/ep2/bench_${cfg}_ep2.err
  tail -c 1500 gpurun_out/ep2/bench_${cfg}_ep2.json; tail -3 gpurun_out/ep2/bench_${cfg}_ep2.err
done
