# bench lines after the grouped weight-gradient walk + transformer launch list with DRAM bytes
mkdir -p gpurun_out/r3y
make -s -j8 all 2>&1 | tail -2
line() {
  python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$2', round(d['value']), round(d['ms_per_step'], 3), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'], 3), d['detail']['per_call_ms'].get('expert_ffn_bwd'), d['clocks'])"
}
python bench.py --steps 20 --warmup 5 > gpurun_out/r3y/bench_transformer.json 2> gpurun_out/r3y/bench_transformer.err; line gpurun_out/r3y/bench_transformer.json transformer
python bench.py --config grid3d --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r3y/bench_grid3d.json 2> gpurun_out/r3y/bench_grid3d.err; line gpurun_out/r3y/bench_grid3d.json grid3d
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/r3y/launches_transformer.csv python tools/profile_step.py --config transformer --steps 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/r3y/launches_transformer.csv > gpurun_out/r3y/launches_transformer.txt; grep "1, 1, 4\|total" gpurun_out/r3y/launches_transformer.txt
python tools/traffic.py gpurun_out/r3y/launches_transformer.csv transformer gpurun_out/r3y/traffic_transformer.json | grep ffn
