#!/bin/bash
cd "$(dirname "$0")/.."
echo "== parity E"; PKV_K3_E=1 timeout 120 python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -1
for rep in 1 2 3; do
for e in 0 1; do
  echo "E=$e rep $rep $(PKV_K3_E=$e timeout 90 python tools/bench_prefill.py --n 2048,4096,8192,16384 2>&1 | tail -4 | python -c "import sys,json; print([round(json.loads(l)['tflops']) for l in sys.stdin])")"
done
done
echo "gathered E=1 $(PKV_K3_E=1 timeout 90 python tools/bench_prefill.py --gathered --n 8192,16384 2>&1 | tail -2 | python -c "import sys,json; print([round(json.loads(l)['tflops']) for l in sys.stdin])")"
