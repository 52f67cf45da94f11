#!/bin/bash
# Alternating sustained A/B of two lags (pieces): bash tools/lag_ab.sh 3 4 [reps]
A=$1; B=$2; N=${3:-4}
for rep in $(seq 1 $N); do
  for L in $A $B; do
    printf 'lag %s ' "$L"
    DVLA_FUSED_LAG=$L python bench.py --steps 200 --warmup 20 --no-e2e --no-cpu --no-repl \
      --no-swimlane --no-gauss --no-f32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); c=d['clocks']; print(round(d['ms_per_step'],4), d['roofline']['kernel_ms'], c['sm_mhz'])"
  done
done
