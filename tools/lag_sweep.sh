#!/bin/bash
# Sustained (power-capped) C2 step time vs the fused kernel's lag (pieces).
for rep in 1 2; do
  for L in "$@"; do
    printf 'lag %s ' "$L"
    DVLA_FUSED_LAG=$L python bench.py --steps 200 --warmup 20 --no-e2e --no-cpu --no-repl \
      --no-swimlane --no-gauss --no-f32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); c=d['clocks']; print(round(d['ms_per_step'],4), d['roofline']['kernel_ms'], d['roofline']['frac'], c['sm_mhz'], c['reasons'], c.get('power_w'))"
  done
done
