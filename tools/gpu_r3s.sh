# 2D operand boxes restored: ffn/sgd parity + full transformer launch list with DRAM bytes
mkdir -p gpurun_out/r3s
make -s -j8 all 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_sgd.py tests/test_gpu_host_step.py -m gpu -q -x --timeout 600 > gpurun_out/r3s/pytest.txt 2>&1; tail -2 gpurun_out/r3s/pytest.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_tc_gemm -c 14 --csv --log-file gpurun_out/r3s/l_full.csv python tools/profile_step.py --config transformer --steps 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r3s/l_full.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); out.setdefault(d["ID"], {"k": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = d["Metric Value"]
for i, m in list(out.items())[-7:]: print(m)
PY
