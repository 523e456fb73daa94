#!/bin/bash
# dW2 GEMM alone (DMOE_BWD_ONLY=4) with parts of its pipeline disabled (DMOE_TC_DEBUG_SEGK:
# 1 no stores, 2 no TMEM loads, 4 no MMAs, 32 no cache hints); per-call expert_ffn_bwd time.
for cfg in ${CFGS:-mnist}; do
  st=400; [ $cfg = transformer ] && st=20
  for f in 0 1 2 4 6 7 32; do
    DMOE_BWD_ONLY=4 DMOE_TC_DEBUG_SEGK=$f python bench.py --config $cfg --steps $st > gpurun_out/segk_${cfg}_$f.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/segk_${cfg}_$f.json').read().strip().splitlines()[-1])
print('$cfg dbg $f dW2 %.4f ms' % d['detail']['per_call_ms']['expert_ffn_bwd'])"
  done
done
