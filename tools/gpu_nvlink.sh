# NVLink data counters around an expert-parallel bench run (2 GPUs): bytes moved per step vs the exchange's rows
mkdir -p gpurun_out/nvl
make -s -j8 all 2>&1 | tail -2
nvidia-smi nvlink -gt d > gpurun_out/nvl/before.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 \
  bench.py --gpus 2 --config transformer --steps 20 --warmup 4 --no-cpu-baseline > gpurun_out/nvl/bench.json 2> gpurun_out/nvl/bench.err
nvidia-smi nvlink -gt d > gpurun_out/nvl/after.txt 2>&1
head -30 gpurun_out/nvl/after.txt
python - <<'PY'
import re
def parse(p):
    tot = {}
    gpu = None
    for line in open(p):
        m = re.match(r"GPU (\d+):", line)
        if m: gpu = int(m.group(1)); continue
        m = re.search(r"Link (\d+): Data Tx: (\d+) KiB", line)
        if m and gpu is not None: tot[(gpu, "tx", int(m.group(1)))] = int(m.group(2))
        m = re.search(r"Link (\d+): Data Rx: (\d+) KiB", line)
        if m and gpu is not None: tot[(gpu, "rx", int(m.group(1)))] = int(m.group(2))
    return tot
b, a = parse("gpurun_out/nvl/before.txt"), parse("gpurun_out/nvl/after.txt")
for g in sorted({k[0] for k in a}):
    tx = sum(a[k] - b.get(k, 0) for k in a if k[0] == g and k[1] == "tx")
    rx = sum(a[k] - b.get(k, 0) for k in a if k[0] == g and k[1] == "rx")
    print(f"GPU {g}: NVLink data tx {tx / 2**20:.2f} GiB, rx {rx / 2**20:.2f} GiB over the whole bench run")
PY
