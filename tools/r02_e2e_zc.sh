#!/bin/bash
# e2e C2: default (q by DMA, k/v zero-copy) vs PKV_ZERO_COPY_IN=1 (q/k/v read through mapped pointers)
cd "$(dirname "$0")/.."
e2e() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['e2e']['value'], round(d['e2e']['ms_per_step']*1e3,1))"; }
for rep in 1 2 3; do
  echo "default $(timeout 200 python bench.py --no-cpu-baseline --no-prefill --no-c5 --no-check --steps 20 --warmup 5 2>/dev/null | e2e)"
  echo "zc_in   $(PKV_ZERO_COPY_IN=1 timeout 200 python bench.py --no-cpu-baseline --no-prefill --no-c5 --no-check --steps 20 --warmup 5 2>/dev/null | e2e)"
done
