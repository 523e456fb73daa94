# beam search tile size A/B: tokens per CTA 128 (2 CTAs/SM) vs 64 (4 CTAs/SM) vs 32 (8 CTAs/SM)
mkdir -p gpurun_out/r4d
for v in "128 2" "64 4" "32 8"; do set -- $v
  make -s clean && make -s -j8 all XFLAGS="-DDMOE_BEAM_TOK=$1 -DDMOE_BEAM_MINB=$2" 2>&1 | tail -2
  timeout 900 python -m pytest tests/test_gpu_routing.py -m gpu -q -x --timeout 600 > gpurun_out/r4d/pytest_$1.txt 2>&1; echo "$1: $(tail -1 gpurun_out/r4d/pytest_$1.txt)"
  for c in transformer grid3d; do
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:beam_topk -c 2 --csv --log-file gpurun_out/r4d/l_$1_$c.csv python tools/profile_step.py --config $c --steps 2 > /dev/null 2>&1
    echo "$1 $c $(grep gpu__time gpurun_out/r4d/l_$1_$c.csv | awk -F'","' '{print $NF}' | tr '\n' ' ')"
  done
done
make -s clean && make -s -j8 all 2>&1 | tail -2
