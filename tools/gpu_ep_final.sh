# final multi-GPU session (4 GPUs): EP parity, per-phase times, EP bench lines at 4 and 2 GPUs
mkdir -p gpurun_out/epf
make -s -j8 all 2>&1 | tail -2
nvidia-smi topo -m > gpurun_out/epf/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ep.py -m gpu -v --timeout 600 > gpurun_out/epf/pytest_ep.txt 2>&1; tail -3 gpurun_out/epf/pytest_ep.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29553 tools/ep_phases.py transformer > gpurun_out/epf/phases_transformer_ep4.txt 2>&1
grep -A15 "rank 0" gpurun_out/epf/phases_transformer_ep4.txt
for n in 4 2; do
for cfg in transformer mnist; do
  st=10; [ $cfg = mnist ] && st=200
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29554 \
    bench.py --gpus $n --config $cfg --steps $st --warmup 4 > gpurun_out/epf/bench_${cfg}_ep$n.json 2> gpurun_out/epf/bench_${cfg}_ep$n.err
  python -c "
import json;d=json.loads(open('gpurun_out/epf/bench_${cfg}_ep$n.json').read().strip().splitlines()[-1]);print('$cfg', $n, round(d['value']),round(d['ms_per_step'],3),round(d['e2e']['value']),d['clocks'])"
done
done
