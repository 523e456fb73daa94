# two rows per warp iteration in the peer exchange: EP parity (2 GPUs), phases at 4 GPUs, EP bench lines at 4 and 2 GPUs
mkdir -p gpurun_out/ep4d
make -s -j8 all 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_ep.py -m gpu -v --timeout 600 > gpurun_out/ep4d/pytest_ep.txt 2>&1; tail -3 gpurun_out/ep4d/pytest_ep.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543 tools/ep_phases.py transformer > gpurun_out/ep4d/phases_transformer_ep4.txt 2>&1
grep -A15 "rank 0" gpurun_out/ep4d/phases_transformer_ep4.txt
for n in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29544 \
    bench.py --gpus $n --config transformer --steps 10 --warmup 4 > gpurun_out/ep4d/bench_transformer_ep$n.json 2> gpurun_out/ep4d/bench_transformer_ep$n.err
  python -c "
import json;d=json.loads(open('gpurun_out/ep4d/bench_transformer_ep$n.json').read().strip().splitlines()[-1]);print($n, d['value'],d['ms_per_step'],d['e2e']['value'],d['clocks'])"
done
