# fix-up warp zeroing with shared stores: parity + launch lists + bench
mkdir -p gpurun_out/r3o
make -s -j8 all 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_sgd.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 > gpurun_out/r3o/pytest.txt 2>&1; tail -2 gpurun_out/r3o/pytest.txt
for v in "k64:M=16 T=4096" "k256:M=32" "full:M=64"; do n=${v%%:*}; a=${v#*:}
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tc_gemm -c 14 --csv --log-file gpurun_out/r3o/l_$n.csv python tools/profile_step.py --config transformer --steps 2 --set $a > /dev/null 2>&1
python - $n <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r3o/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r != hdr]
for d in out[-7:]: print(sys.argv[1], d["Kernel Name"].split("(")[0][:40], round(float(d["Metric Value"]) / 1000, 1), "us")
PY
done
python bench.py --steps 5 --warmup 3 > gpurun_out/r3o/bench.json 2> gpurun_out/r3o/bench.err; python -c "
import json;d=json.loads(open('gpurun_out/r3o/bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['detail']['per_call_ms'],d['clocks'])"
