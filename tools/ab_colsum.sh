python tools/hbm_probe.py
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export DMOE_NO_COLSUM_FUSE=1; else unset DMOE_NO_COLSUM_FUSE; fi
  python bench.py --config transformer --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nofuse=$v', round(d['ms_per_step'],3), round(d['detail']['per_call_ms']['expert_ffn_bwd'],3), d['clocks'])"
done
