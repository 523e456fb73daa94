# grouped weight-gradient walk: parity + dW GEMM time / DRAM reads (transformer, M=32, grid3d) + bench
mkdir -p gpurun_out/r3v
make -s -j8 all 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_sgd.py tests/test_gpu_parity.py tests/test_gpu_ffn3.py tests/test_gpu_host_step.py -m gpu -q -x --timeout 600 > gpurun_out/r3v/pytest.txt 2>&1; tail -2 gpurun_out/r3v/pytest.txt
lst() {
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_tc_gemm -c 16 --csv --log-file gpurun_out/r3v/l_$1.csv python tools/profile_step.py --config $2 --steps 2 $3 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r3v/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); out.setdefault(d["ID"], {"k": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = d["Metric Value"]
for i, m in list(out.items())[-7:]:
    if ", 1, 1, " in m["k"]: print(sys.argv[1], m["k"], round(float(m["gpu__time_duration.sum"]) / 1e3, 1), "us", round(float(m["dram__bytes_read.sum"]) / 1e9, 2), "GB read")
PY
}
lst transformer transformer ""
lst m32 transformer "--set M=32"
lst grid3d grid3d ""
python bench.py --steps 10 --warmup 3 > gpurun_out/r3v/bench.json 2> gpurun_out/r3v/bench.err; python -c "
import json;d=json.loads(open('gpurun_out/r3v/bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['detail']['per_call_ms']['expert_ffn_bwd'],d['clocks'])"
