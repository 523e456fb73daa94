# ring depth 2 vs 3 with the grouped walk (transformer dW GEMM, EXPERIMENTS build, same box)
mkdir -p gpurun_out/r4f
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
lst() {
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_tc_gemm" -c 16 --csv --log-file gpurun_out/r4f/l_$1.csv python tools/profile_step.py --config transformer --steps 2 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r4f/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); out.setdefault(d["ID"], {"k": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = d["Metric Value"]
for i, m in list(out.items())[-7:]:
    if ", 1, 1, 4" in m["k"]: print(sys.argv[1], round(float(m["gpu__time_duration.sum"]) / 1e3, 1), "us", round(float(m["dram__bytes_read.sum"]) / 1e9, 2), "GB read")
PY
}
for r in 1 2; do lst s3_$r; DMOE_TC_STAGES=2 lst s2_$r; DMOE_TC_STAGES=1 lst s1_$r; done
make -s clean && make -s -j8 all 2>&1 | tail -2
