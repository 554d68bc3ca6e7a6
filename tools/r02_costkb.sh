#!/bin/bash
# decode planner per-item cost sweep (PKV_DECODE_COST_KB): C2, C5, C3 points
for kb in 600 400 300 250 200; do
  for rep in 1 2; do
    c2=$(PKV_DECODE_COST_KB=$kb timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-prefill --no-c5 --no-check --steps 20 --warmup 5 | python -c "import json,sys; print(json.load(sys.stdin)['value'])")
    echo "kb=$kb rep=$rep c2=$c2"
  done
  c5=$(PKV_DECODE_COST_KB=$kb timeout 300 python bench.py --config c5 --no-cpu-baseline --no-e2e --no-prefill --no-check --steps 10 --warmup 3 | python -c "import json,sys; print(json.load(sys.stdin)['value'])")
  c3a=$(PKV_DECODE_COST_KB=$kb timeout 120 python bench.py --config c3 --context 4096 --batch 32 --no-cpu-baseline --no-e2e --no-prefill --no-check --steps 10 --warmup 3 | python -c "import json,sys; print(json.load(sys.stdin)['value'])")
  c3b=$(PKV_DECODE_COST_KB=$kb timeout 120 python bench.py --config c3 --context 16384 --batch 8 --no-cpu-baseline --no-e2e --no-prefill --no-check --steps 10 --warmup 3 | python -c "import json,sys; print(json.load(sys.stdin)['value'])")
  echo "kb=$kb c5=$c5 c3_4kx32=$c3a c3_16kx8=$c3b"
done
