#!/bin/bash
# small-batch decode step / launch times (planner's choice), B = 1 / 4 / 8
for a in "1 2048" "1 8192" "1 32768" "4 2048" "4 8192" "4 32768" "8 8192"; do
  set -- $a
  python bench.py --config c3 --batch $1 --context $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-prefill --no-check 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('B=$1 ctx=$2 step %.1f us kernel %.1f us %.0f GB/s' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms_mean']*1e3, d['value']))"
done
