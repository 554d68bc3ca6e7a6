#!/bin/bash
# K3 exp2 share on the FMA pipe: in-tree (1 of 8 pairs) vs variant builds
cd "$(dirname "$0")/.."
V=paper_2506_07311_b200/variants
echo "parity: $(timeout 120 python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -1)"
for rep in 1 2; do
  for name in product emu1p32 emu2p32 emu3p32; do
    lib=$V/lib_$name.so; [ $name = product ] && lib=paper_2506_07311_b200/libpkv200.so
    echo "$name $(PKV200_LIB=$lib timeout 90 python tools/bench_prefill.py --n 2048,4096,8192,16384 2>&1 | tail -4 | python -c "import sys,json; print([round(json.loads(l)['tflops']) for l in sys.stdin])")"
  done
done
