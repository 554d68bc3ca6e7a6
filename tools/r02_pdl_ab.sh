#!/bin/bash
# A/B: decode launch with programmatic dependent launch behind the step's aux kernel (PKV_DECODE_PDL)
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
e2e() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], round(d['e2e']['ms_per_step']*1e3,1))"; }
for rep in 1 2 3; do
  for pdl in 0 1; do
    echo "pdl=$pdl $(PKV_DECODE_PDL=$pdl timeout 200 python bench.py --no-cpu-baseline --no-prefill --no-c5 --no-check --steps 30 --warmup 5 2>/dev/null | e2e)"
  done
done
for pdl in 0 1; do
  echo "c3 b=4 8k pdl=$pdl $(PKV_DECODE_PDL=$pdl timeout 200 python bench.py --config c3 --context 8192 --batch 4 --no-cpu-baseline --no-prefill --no-check --steps 20 --warmup 5 2>/dev/null | e2e)"
done
