# gate-backward dx kernel occupancy variants (UNR, min blocks per SM): launch lists at transformer / grid3d
mkdir -p gpurun_out/r4a
for v in "4 1" "2 5" "2 4"; do set -- $v
  make -s clean && make -s -j8 all XFLAGS="-DGBDX_UNR4=$1 -DGBDX_MINB=$2" 2>&1 | tail -2
  for c in transformer grid3d; do
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gate_bwd_dx -c 2 --csv --log-file gpurun_out/r4a/l_$1_$2_$c.csv python tools/profile_step.py --config $c --steps 2 > /dev/null 2>&1
    echo "$1 $2 $c $(grep gpu__time gpurun_out/r4a/l_$1_$2_$c.csv | tail -1 | awk -F'","' '{print $NF}')"
  done
done
make -s clean && make -s -j8 all 2>&1 | tail -2
