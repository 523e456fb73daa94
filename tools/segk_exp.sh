# weight-gradient GEMM experiments (EXPERIMENTS build on the box only): kernel time per variant on
# a transformer-shaped slice (256 experts x 64 rows, D 1024, H 4096) from an ncu launch list
mkdir -p gpurun_out/segk
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
for v in "base:" "nostore:DMOE_TC_DEBUG_SEGK=1" "nomma:DMOE_TC_DEBUG_SEGK=4" "noload_tmem:DMOE_TC_DEBUG_SEGK=2" "bn128:DMOE_TC_BN=128" "noL2hint:DMOE_TC_DEBUG_SEGK=32"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:k_tc_gemm --csv \
    --log-file gpurun_out/segk/$name.csv python tools/profile_step.py --config transformer --steps 1 --set M=16 T=4096 > /dev/null 2>&1
  python - "$name" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/segk/{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = {}
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0]
        out.setdefault(k, {})[d["Metric Name"]] = d["Metric Value"]
for k, m in out.items():
    if "1, 1" in k or "true, true" in k:
        print(sys.argv[1], k[:40], m)
PY
done
make -s clean && make -s -j8 all 2>&1 | tail -2
