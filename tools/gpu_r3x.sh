# L2-sized expert groups for the weight-gradient walk: parity (product build) + A/B of the group size (EXPERIMENTS build)
mkdir -p gpurun_out/r3x
make -s -j8 all 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_sgd.py tests/test_gpu_parity.py tests/test_gpu_ffn3.py tests/test_gpu_host_step.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 900 > gpurun_out/r3x/pytest.txt 2>&1; tail -2 gpurun_out/r3x/pytest.txt
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
lst() {
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_tc_gemm -c 16 --csv --log-file gpurun_out/r3x/l_$1.csv python tools/profile_step.py --config $2 --steps 2 $3 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r3x/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); out.setdefault(d["ID"], {"k": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = d["Metric Value"]
for i, m in list(out.items())[-7:]:
    if ", 1, 1, 4" in m["k"]: print(sys.argv[1], m["k"], round(float(m["gpu__time_duration.sum"]) / 1e3, 1), "us", round(float(m["dram__bytes_read.sum"]) / 1e9, 2), "GB read")
PY
}
for g in auto 1 4; do
  if [ $g = auto ]; then unset DMOE_SEGK_GS; else export DMOE_SEGK_GS=$g; fi
  lst tf_$g transformer ""
  lst g3_$g grid3d ""
  lst m16_$g transformer "--set M=16"
done
unset DMOE_SEGK_GS
make -s clean && make -s -j8 all 2>&1 | tail -2
