#!/bin/bash
# weight-gradient GEMMs alone (DMOE_BWD_ONLY=12) with / without the L2 prefetch cursor (flag 16)
for cfg in ${CFGS:-mnist transformer}; do
  st=400; [ $cfg = transformer ] && st=20
  for f in 0 16; do
    DMOE_BWD_ONLY=12 DMOE_TC_DEBUG_SEGK=$f python bench.py --config $cfg --steps $st > gpurun_out/pf_${cfg}_$f.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/pf_${cfg}_$f.json').read().strip().splitlines()[-1])
print('$cfg segk flags $f dW2+dW1 %.4f ms' % d['detail']['per_call_ms']['expert_ffn_bwd'])"
  done
done
