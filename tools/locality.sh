#!/bin/bash
run() { python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', d['value'], round(d['roofline']['k2_ms_mean']*1000,1), 'us')" 2>/dev/null || echo "$* FAILED"; }
run --waves 1
run --config c3 --context 8192 --batch 64 --waves 1
run --config c3 --context 2048 --batch 64 --heads 32:32 --waves 1
run --config c3 --context 8192 --batch 64 --heads 8:8 --waves 1
run --config c3 --context 8192 --batch 16 --heads 32:32 --waves 1
run --config c3 --context 2048 --batch 128 --heads 16:16 --waves 1
run --config c3 --context 8192 --batch 128 --heads 8:4 --waves 1
