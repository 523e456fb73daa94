# weight-gradient walk A/B/C on one box: strided / grouped interleaved / grouped contiguous (EXPERIMENTS build)
mkdir -p gpurun_out/r3w
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
lst() {
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_tc_gemm -c 16 --csv --log-file gpurun_out/r3w/l_$1.csv python tools/profile_step.py --config $2 --steps 2 $3 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r3w/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); out.setdefault(d["ID"], {"k": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = d["Metric Value"]
for i, m in list(out.items())[-7:]:
    if ", 1, 1, 4" in m["k"]: print(sys.argv[1], m["k"], round(float(m["gpu__time_duration.sum"]) / 1e3, 1), "us", round(float(m["dram__bytes_read.sum"]) / 1e9, 2), "GB read")
PY
}
for w in 0 1 2; do
  DMOE_SEGK_WALK=$w lst tf_w$w transformer ""
  DMOE_SEGK_WALK=$w lst g3_w$w grid3d ""
done
for w in 0 1 2; do DMOE_SEGK_WALK=$w lst tf2_w$w transformer ""; done
make -s clean && make -s -j8 all 2>&1 | tail -2
