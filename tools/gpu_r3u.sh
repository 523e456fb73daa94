# full-size dW GEMM: ring depth 2 vs 3, and 128-wide tiles (two launches, 4 stages) (EXPERIMENTS build, no debug flags)
mkdir -p gpurun_out/r3u
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
lst() {
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_tc_gemm -c 16 --csv --log-file gpurun_out/r3u/l_$1.csv python tools/profile_step.py --config transformer --steps 2 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r3u/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); out.setdefault(d["ID"], {"k": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = d["Metric Value"]
for i, m in list(out.items())[-8:]:
    if ", 1, 1, 4" in m["k"]: print(sys.argv[1], m)
PY
}
lst base
DMOE_TC_STAGES=2 lst stages2
DMOE_TC_BN=128 lst bn128
make -s clean && make -s -j8 all 2>&1 | tail -2
