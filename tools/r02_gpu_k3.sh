#!/bin/bash
cd "$(dirname "$0")/.."
echo "== parity"; timeout 120 python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -3
echo "== paged"; timeout 90 python tools/bench_prefill.py --n 2048,4096,8192,16384 2>&1 | tail -4
echo "== gathered"; timeout 90 python tools/bench_prefill.py --gathered --n 8192,16384 2>&1 | tail -2
echo "== timeline"; PF_DEBUG=1 timeout 60 python tools/bench_prefill.py --n 8192 2>&1 | head -9
