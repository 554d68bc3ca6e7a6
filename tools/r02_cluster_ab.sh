#!/bin/bash
# small-batch decode: forced cluster sizes (PKV_DECODE_CLUSTER; unset = planner), step and kernel times
for cl in "" 1 2 4 8 16; do
  for a in "1 2048" "1 32768" "4 8192"; do
    set -- $a
    PKV_DECODE_CLUSTER=$cl timeout 60 python bench.py --config c3 --batch $1 --context $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-prefill --no-check --no-c5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('cluster=${cl:-auto} B=$1 ctx=$2 step %.1f us kernel %.1f us %.0f GB/s' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms_mean']*1e3, d['value']))"
  done
done
