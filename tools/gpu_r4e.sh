# tensor-pipe utilisation of the tcgen05 GEMMs at grid3d and transformer (ncu metrics, one eager step)
mkdir -p gpurun_out/r4e
make -s -j8 all 2>&1 | tail -2
for c in grid3d transformer; do
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_tc_gemm -c 14 --csv --log-file gpurun_out/r4e/tensor_$c.csv python tools/profile_step.py --config $c --steps 2 > /dev/null 2>&1
python - $c <<'PY'
import csv, sys
c = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/r4e/tensor_{c}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); out.setdefault(d["ID"], {"k": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = d["Metric Value"]
print(f"# {c}: tcgen05 GEMM launches of one step (ncu, cold, serialised, --clock-control none)")
print("kernel | ms | tensor pipe active % of peak | SM clock GHz | DRAM read GB | DRAM write GB")
for i, m in list(out.items())[-7:]:
    print(m["k"].replace("void ", ""), "|", round(float(m["gpu__time_duration.sum"]) / 1e6, 3), "|",
          m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"], "|",
          round(float(m["sm__cycles_elapsed.avg.per_second"]) / 1e9, 3), "|",
          round(float(m["dram__bytes_read.sum"]) / 1e9, 2), "|", round(float(m["dram__bytes_write.sum"]) / 1e9, 2))
PY
done
