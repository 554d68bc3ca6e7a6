#!/bin/bash
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests/test_gpu_decode_tc.py tests/test_gpu_step_atomicity.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for rep in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-prefill --no-c5 --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], 'parity', d['parity_checked'])"
done
timeout 200 python tools/e2e_variants.py 2>&1 | tail -5
