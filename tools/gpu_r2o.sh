mkdir -p gpurun_out/r2o
make -s -j8 all 2>&1 | tail -3
for cfg in transformer mnist mnist_block transformer_block grid3d; do
  st=30; [ $cfg = mnist ] && st=300; [ $cfg = mnist_block ] && st=300; [ $cfg = grid3d ] && st=10
  nc=""; [ $cfg != transformer ] && nc="--no-cpu-baseline"
  timeout 900 python bench.py --config $cfg --steps $st $nc > gpurun_out/r2o/bench_$cfg.json 2> gpurun_out/r2o/bench_$cfg.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2o/bench_$cfg.json').read().strip().splitlines()[-1])
print('$cfg', round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])
print('  ', {k: round(v,3) for k,v in d['detail']['per_call_ms'].items()})" || tail -3 gpurun_out/r2o/bench_$cfg.err
done
bash tools/sanitize.sh
