# after the shared-store zeroing: skeleton vs real at full size + role waits (EXPERIMENTS build)
mkdir -p gpurun_out/r3p
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
lst() {
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tc_gemm -c 14 --csv --log-file gpurun_out/r3p/l_$1.csv python tools/profile_step.py --config transformer --steps 2 --set $2 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r3p/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r != hdr]
for d in out[-7:]:
    if "1, 1, 4" in d["Kernel Name"]: print(sys.argv[1], d["Kernel Name"].split("(")[0][:40], round(float(d["Metric Value"]) / 1000, 1), "us")
PY
}
lst base_full "M=64"
DMOE_TC_DEBUG_SEGK=519 lst skeleton_full "M=64"
DMOE_TC_DEBUG_SEGK=7 lst nothing_full "M=64"
python tools/tc_wait.py transformer > gpurun_out/r3p/wait_full.txt 2>&1
DMOE_TC_DEBUG_SEGK=519 python tools/tc_wait.py transformer > gpurun_out/r3p/wait_skel_full.txt 2>&1
grep -A6 "SEGK=1, EPI=4" gpurun_out/r3p/wait_*.txt
make -s clean && make -s -j8 all 2>&1 | tail -2
