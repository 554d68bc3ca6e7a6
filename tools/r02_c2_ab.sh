#!/bin/bash
# C2 device value A/B: $A_LIB vs the in-tree library, alternating, 3 reps
cd "$(dirname "$0")/.."
val() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'])"; }
for rep in 1 2 3; do
  for lib in "$A_LIB" paper_2506_07311_b200/libpkv200.so; do
    echo "$(basename $lib) $(PKV200_LIB=$lib timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-prefill --no-c5 --steps 20 --warmup 5 2>/dev/null | val)"
  done
done
