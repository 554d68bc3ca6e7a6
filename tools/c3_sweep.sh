#!/bin/bash
# C3 decode sweep (Llama-3-8B GQA 32q/8kv x128 bf16, page 16): KV GB/s and
# per-step time vs context and batch; one bench.py process per point.
for ctx in 2048 4096 8192 16384 32768; do
  for b in 1 2 4 8 16 32 64; do
    python bench.py --config c3 --context $ctx --batch $b --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-prefill 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ctx=%d batch=%d %.1f GB/s %.1f %% %.1f us/step %.0f tok/s' % ($ctx, $b, d['value'], d['pct_of_8TBs'], d['ms_per_step']*1e3, d['tokens_per_s']))"
  done
done
