#!/bin/bash
# A/B of the decode planner's minimum piece (PKV_DECODE_ITEM_KB) on C2 / C5 / C3 points
cd "$(dirname "$0")/.."
val() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'])"; }
B="--no-cpu-baseline --no-e2e --no-prefill --no-c5 --no-check --steps 30 --warmup 5"
for rep in 1 2 3; do
  for kb in 400 256 128; do
    echo "c2 kb=$kb $(PKV_DECODE_ITEM_KB=$kb timeout 120 python bench.py $B | val)"
  done
done
for kb in 400 256; do
  echo "c5 kb=$kb $(PKV_DECODE_ITEM_KB=$kb timeout 300 python bench.py --config c5 $B | val)"
  echo "c3 16x8k kb=$kb $(PKV_DECODE_ITEM_KB=$kb timeout 120 python bench.py --config c3 --context 8192 --batch 16 $B | val)"
  echo "c3 64x2k kb=$kb $(PKV_DECODE_ITEM_KB=$kb timeout 120 python bench.py --config c3 --context 2048 --batch 64 $B | val)"
done
