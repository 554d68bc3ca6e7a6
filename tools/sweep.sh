#!/bin/bash
# quick decode bandwidth sweep: prints config, GB/s, K2 ms
run() { python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', d['value'], round(d['roofline']['k2_ms_mean']*1000,1), 'us')" 2>/dev/null || echo "$* FAILED"; }
for w in 0; do
  run 
  for b in 1 4 16 64; do run --config c3 --context 8192 --batch $b ; done
  run --config c3 --context 32768 --batch 8 
done
