# weight-gradient tail boxes: parity (product build) + same-box A/B with / without (EXPERIMENTS build)
mkdir -p gpurun_out/r4b
make -s clean && make -s -j8 all 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_sgd.py tests/test_gpu_parity.py tests/test_gpu_ffn3.py tests/test_gpu_host_step.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 900 > gpurun_out/r4b/pytest.txt 2>&1; tail -2 gpurun_out/r4b/pytest.txt
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
lst() {
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_tc_gemm|gate_bwd_dx" -c 20 --csv --log-file gpurun_out/r4b/l_$1.csv python tools/profile_step.py --config $2 --steps 2 $3 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r4b/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); out.setdefault(d["ID"], {"k": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = d["Metric Value"]
for i, m in list(out.items())[-8:]:
    if ", 1, 1, 4" in m["k"] or "gate_bwd_dx" in m["k"]: print(sys.argv[1], m["k"][:45], round(float(m["gpu__time_duration.sum"]) / 1e3, 1), "us", round(float(m["dram__bytes_read.sum"]) / 1e9, 2), "GB read")
PY
}
for r in 1 2; do
  lst tail_tf$r transformer ""
  DMOE_TC_NOTAIL=1 lst notail_tf$r transformer ""
done
lst tail_g3 grid3d ""
DMOE_TC_NOTAIL=1 lst notail_g3 grid3d ""
make -s clean && make -s -j8 all 2>&1 | tail -2
