#!/bin/bash
# Alternating sustained A/B of library variants: bash tools/variant_ab.sh N default a.so b.so
N=$1; shift
for rep in $(seq 1 $N); do
  for v in "$@"; do
    if [ "$v" = default ]; then L=""; else L=$v; fi
    printf '%s ' "$(basename "$v")"
    DVLA_B200_LIB=$L python bench.py --steps 200 --warmup 20 --no-e2e --no-cpu --no-repl \
      --no-swimlane --no-gauss --no-f32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); c=d['clocks']; print(round(d['ms_per_step'],4), d['roofline']['kernel_ms'], c['sm_mhz'])"
  done
done
