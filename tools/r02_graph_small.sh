#!/bin/bash
# e2e A/B of the CUDA-graph step mode (PKV_STEP_GRAPH) on small C3 batches and C2
cd "$(dirname "$0")/.."
e2e() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['e2e']['value'], round(d['e2e']['ms_per_step']*1e3,1))"; }
for pt in 1:2048 1:32768 4:8192 16:8192; do
  b=${pt%%:*}; c=${pt##*:}
  for rep in 1 2; do
    for g in 0 1; do
      echo "b=$b ctx=$c graph=$g $(PKV_STEP_GRAPH=$g timeout 200 python bench.py --config c3 --context $c --batch $b --no-cpu-baseline --no-prefill --no-check --steps 30 --warmup 5 2>/dev/null | e2e)"
    done
  done
done
for g in 0 1; do echo "c2 graph=$g $(PKV_STEP_GRAPH=$g timeout 200 python bench.py --no-cpu-baseline --no-prefill --no-c5 --no-check --steps 30 --warmup 5 2>/dev/null | e2e)"; done
