#!/bin/bash
# C3 4 x 8k e2e: per-step wall times around the mirror's column doubling (512 -> 1024 pages), lazy vs eager module loading
cd "$(dirname "$0")/.."
for ml in LAZY EAGER; do
  echo "CUDA_MODULE_LOADING=$ml"
  CUDA_MODULE_LOADING=$ml PKV_E2E_STEP_TIMES=1 timeout 200 python bench.py --config c3 --context 8192 --batch 4 --no-cpu-baseline --no-prefill --no-check --steps 20 --warmup 5 2>&1 | grep -E 'e2e step|^\{' | cut -c1-300
done
