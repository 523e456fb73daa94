# transformer dW GEMM: tail rows 16 vs 32, group sizes 2 / 4 / 8 (EXPERIMENTS build, same box)
mkdir -p gpurun_out/r4c
lst() {
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_tc_gemm" -c 16 --csv --log-file gpurun_out/r4c/l_$1.csv python tools/profile_step.py --config transformer --steps 2 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r4c/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); out.setdefault(d["ID"], {"k": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = d["Metric Value"]
for i, m in list(out.items())[-7:]:
    if ", 1, 1, 4" in m["k"]: print(sys.argv[1], round(float(m["gpu__time_duration.sum"]) / 1e3, 1), "us", round(float(m["dram__bytes_read.sum"]) / 1e9, 2), "GB read")
PY
}
for t in 32 16; do
  make -s clean && make -s -j8 all EXPERIMENTS=1 XFLAGS="-DDMOE_TAIL_ROWS=$t" 2>&1 | tail -2
  lst tail$t
  for g in 2 8; do DMOE_SEGK_GS=$g lst tail${t}_gs$g; done
  lst tail${t}_again
done
make -s clean && make -s -j8 all 2>&1 | tail -2
