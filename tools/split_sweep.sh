#!/bin/bash
# Sweep the expert-backward SM split (DMOE_BWD_SEGK_CTAS) on mnist and transformer.
mkdir -p gpurun_out
for c in ${CTAS:-0 40 56 74 92}; do
  for cfg in ${CFGS:-mnist transformer}; do
    st=400; [ $cfg = transformer ] && st=20
    DMOE_BWD_SEGK_CTAS=$c python bench.py --config $cfg --steps $st > gpurun_out/split_${cfg}_$c.json 2>/dev/null
    python - "$cfg" "$c" gpurun_out/split_${cfg}_$c.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
pc = d["detail"]["per_call_ms"]
print(f"{sys.argv[1]:12s} segk_ctas={sys.argv[2]:>3s} step {d['ms_per_step']:.3f} ms  ffn_bwd {pc['expert_ffn_bwd']:.3f}  ffn_fwd {pc['expert_ffn_fwd']:.3f}  clk {d['clocks']['sm_mhz']}")
PY
  done
done
