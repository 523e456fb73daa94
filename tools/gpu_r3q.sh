# host-buffer layer step through the C ABI: test + bench line
mkdir -p gpurun_out/r3q
make -s -j8 all 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_host_step.py tests/test_gpu_ep.py -m gpu -q -x --timeout 600 > gpurun_out/r3q/pytest.txt 2>&1; tail -3 gpurun_out/r3q/pytest.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/r3q/bench.json 2> gpurun_out/r3q/bench.err; tail -3 gpurun_out/r3q/bench.err; python -c "
import json;d=json.loads(open('gpurun_out/r3q/bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e'],d['clocks'])"
python bench.py --config mnist --steps 50 --warmup 5 > gpurun_out/r3q/bench_mnist.json 2> gpurun_out/r3q/bench_mnist.err; python -c "
import json;d=json.loads(open('gpurun_out/r3q/bench_mnist.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e'])"
