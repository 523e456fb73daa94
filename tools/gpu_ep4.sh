# 4-GPU session: expert-parallel parity and EP bench lines at N = 2 and 4 (transformer, mnist)
mkdir -p gpurun_out/ep4
make -s -j8 all 2>&1 | tail -3
nvidia-smi topo -m > gpurun_out/ep4/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ep.py -m gpu -v --timeout 600 > gpurun_out/ep4/pytest_ep.txt 2>&1; tail -8 gpurun_out/ep4/pytest_ep.txt
for n in 4 2; do
for cfg in transformer mnist; do
  st=10; [ $cfg = mnist ] && st=200
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $n --config $cfg --steps $st --warmup 4 > gpurun_out/ep4/bench_${cfg}_ep$n.json 2> gpurun_out/ep4/bench_${cfg}_ep$n.err
  tail -c 400 gpurun_out/ep4/bench_${cfg}_ep$n.json; tail -3 gpurun_out/ep4/bench_${cfg}_ep$n.err
done
done
