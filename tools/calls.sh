#!/bin/bash
# per-ABI-call ms (eager, events) and step for the configs
for cfg in ${CFGS:-mnist transformer}; do
  st=400; [ $cfg != mnist ] && st=20
  python bench.py --config $cfg --steps $st > gpurun_out/calls.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/calls.json').read().strip().splitlines()[-1])
print('$cfg', 'step %.4f' % d['ms_per_step'], {k: round(v, 4) for k, v in d['detail']['per_call_ms'].items()})"
done
