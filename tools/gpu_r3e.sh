# weight-gradient GEMM: L2 prefetch cursor on/off (EXPERIMENTS build)
mkdir -p gpurun_out/r3e
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
lst() {
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_tc_gemm -c 14 --csv --log-file gpurun_out/r3e/l_$1.csv python tools/profile_step.py --config transformer --steps 2 --set $2 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r3e/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); out.setdefault(d["ID"], {})[d["Metric Name"]] = d["Metric Value"]; out[d["ID"]]["k"] = d["Kernel Name"]
for i, m in list(out.items())[-7:]:
    if "1, 1, 4" in m["k"]: print(sys.argv[1], m["k"].split("(")[0][:40], m)
PY
}
lst base_k64 "M=16 T=4096"; lst base_full "M=64"
export DMOE_TC_DEBUG=16
lst pf_k64 "M=16 T=4096"; lst pf_full "M=64"; lst pf_k256 "M=32"
unset DMOE_TC_DEBUG
make -s clean && make -s -j8 all 2>&1 | tail -2
