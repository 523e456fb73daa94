mkdir -p gpurun_out/r2v
make -s -j8 all 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "mnist or tiny or k8 or transformer" > gpurun_out/r2v/pytest.txt 2>&1; tail -2 gpurun_out/r2v/pytest.txt
for c in transformer grid3d; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gate_bwd|gate_reduce" -c 8 --csv --log-file gpurun_out/r2v/launches_$c.csv python tools/profile_step.py --config $c --steps 2 > gpurun_out/r2v/ncu_$c.log 2>&1
grep gpu__time_duration gpurun_out/r2v/launches_$c.csv | cut -c1-40,200-400 | tail -4
done
python bench.py --steps 5 --warmup 3 > gpurun_out/r2v/bench_transformer.json 2> gpurun_out/r2v/bench_transformer.err; tail -c 600 gpurun_out/r2v/bench_transformer.json
ncu --set full --import-source on --clock-control none -k regex:"gate_bwd_dx" -s 1 -c 1 -o gpurun_out/r2v/gbdx_full python tools/profile_step.py --config transformer --steps 2 > gpurun_out/r2v/ncu_full.log 2>&1; tail -1 gpurun_out/r2v/ncu_full.log
