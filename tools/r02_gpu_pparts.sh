#!/bin/bash
cd "$(dirname "$0")/.."
V=paper_2506_07311_b200/variants
echo "== parity 4 parts"; PKV200_LIB=$V/lib_pparts4.so timeout 120 python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -1
for rep in 1 2; do
  for name in pparts1 product pparts4; do
    lib=$V/lib_$name.so; [ $name = product ] && lib=paper_2506_07311_b200/libpkv200.so
    echo "== $name rep $rep"; PKV200_LIB=$lib timeout 90 python tools/bench_prefill.py --n 2048,8192,16384 2>&1 | tail -3 | python -c "import sys,json; print([round(json.loads(l)['tflops']) for l in sys.stdin])"
  done
done
