# full GPU test suite checkpoint + transformer bench
mkdir -p gpurun_out/r3r
make -s -j8 all 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/r3r/pytest_gpu.txt 2>&1; tail -4 gpurun_out/r3r/pytest_gpu.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/r3r/bench.json 2> gpurun_out/r3r/bench.err; python -c "
import json;d=json.loads(open('gpurun_out/r3r/bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['clocks'])"
