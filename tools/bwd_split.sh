#!/bin/bash
# Expert-backward time with subsets of its four GEMMs (DMOE_BWD_ONLY mask: 1 dh, 2 dxd, 4 dW2, 8 dW1).
for cfg in ${CFGS:-mnist}; do
  unset DMOE_SERIAL
  st=400; [ $cfg = transformer ] && st=20
  for m in 1 2 4 8 3 12 15 S; do
    if [ $m = S ]; then export DMOE_SERIAL=1; m=15; fi
    DMOE_BWD_ONLY=$m python bench.py --config $cfg --steps $st > gpurun_out/bwd_${cfg}_$m.json 2>/dev/null
    python -c "
import json,sys; d=json.loads(open('gpurun_out/bwd_${cfg}_$m.json').read().strip().splitlines()[-1])
print('$cfg mask $m ffn_bwd %.4f ms' % d['detail']['per_call_ms']['expert_ffn_bwd'])"
  done
done
