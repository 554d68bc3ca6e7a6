#!/bin/bash
for kb in 350 400 450 500; do
  for rep in 1 2 3; do
    c2=$(PKV_DECODE_COST_KB=$kb timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-prefill --no-c5 --no-check --steps 20 --warmup 5 | python -c "import json,sys; print(json.load(sys.stdin)['value'])")
    echo "kb=$kb rep=$rep c2=$c2"
  done
done
c5=$(PKV_DECODE_COST_KB=400 timeout 300 python bench.py --fragment --no-cpu-baseline --no-e2e --no-prefill --no-c5 --no-check --steps 20 --warmup 5 | python -c "import json,sys; print(json.load(sys.stdin)['value'])"); echo "kb=400 c2frag=$c5"
