#!/bin/bash
# small-batch decode A/B: $A_LIB vs the in-tree library on C3 points (cluster mode), plus the decode tests
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests/test_gpu_decode_tc.py tests/test_gpu_parity.py tests/test_gpu_step_atomicity.py -x -q 2>&1 | tail -1
val() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1), d.get('parity_checked'))"; }
for pt in "1 2048" "1 8192" "4 8192" "8 2048" "4 2048" "16 2048"; do
  set -- $pt
  for lib in "$A_LIB" paper_2506_07311_b200/libpkv200.so; do
    r=""
    for rep in 1 2; do r="$r $(PKV200_LIB=$lib timeout 120 python bench.py --config c3 --batch $1 --context $2 --no-cpu-baseline --no-e2e --no-prefill --no-c5 --steps 20 --warmup 5 2>/dev/null | val)"; done
    echo "B=$1 ctx=$2 $(basename $lib): $r"
  done
done
