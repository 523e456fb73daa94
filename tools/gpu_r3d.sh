# weight-gradient epilogue: LSU stores vs TMA bulk stores
mkdir -p gpurun_out/r3d
make -s -j8 all 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_sgd.py -m gpu -q -x --timeout 600 > gpurun_out/r3d/pytest.txt 2>&1; tail -2 gpurun_out/r3d/pytest.txt
lst() {
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tc_gemm -c 14 --csv --log-file gpurun_out/r3d/l_$1.csv python tools/profile_step.py --config transformer --steps 2 --set $2 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/r3d/l_{sys.argv[1]}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
out = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r != hdr]
for d in out[-7:]:
    if "1, 1, 4" in d["Kernel Name"]: print(sys.argv[1], d["Kernel Name"].split("(")[0][:40], round(float(d["Metric Value"]) / 1000, 1), "us")
PY
}
lst lsu_k64 "M=16 T=4096"; lst lsu_k256 "M=32"; lst lsu_full "M=64"
make -s clean && make -s -j8 all EXPERIMENTS=1 2>&1 | tail -2
export DMOE_TC_DEBUG=256
lst tma_k64 "M=16 T=4096"; lst tma_full "M=64"
unset DMOE_TC_DEBUG
make -s clean && make -s -j8 all 2>&1 | tail -2
