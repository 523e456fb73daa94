#!/bin/bash
# A/B an environment switch on the bench: ENVS="A=1" (empty = baseline), CFGS, REPS
for cfg in ${CFGS:-mnist}; do
  st=400; [ $cfg != mnist ] && st=20
  for rep in $(seq ${REPS:-2}); do
    for e in "" ${ENVS}; do
      env $e python bench.py --config $cfg --steps $st > gpurun_out/ab.json 2>/dev/null
      python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); pc=d['detail']['per_call_ms']
print('%-12s %-24s step %.4f ms  fwd %.4f  bwd %.4f  e2e %.0f' % ('$cfg', '${e:-baseline}', d['ms_per_step'], pc['expert_ffn_fwd'], pc['expert_ffn_bwd'], d['e2e']['value']))"
    done
  done
done
