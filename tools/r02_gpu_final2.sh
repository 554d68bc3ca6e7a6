#!/bin/bash
# round-end pass (re-entry session): GPU suite, smoke, bench + reference arm,
# launch list, ncu --set full of K2-TC (C2) and K3 (8k), memcheck of the new host paths
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/r02_gpu_final.sh
K="--set full --clock-control none --import-source on -k regex:decode_tc -s 2 -c 1 -f"
timeout 400 ncu $K -o gpurun_out/r02_k2_c2_final python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill --no-c5 --no-check > /dev/null 2>&1; echo "ncu k2 rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 3 -c 1 -f -o gpurun_out/r02_k3_final python tools/bench_prefill.py --n 8192 --iters 1 > /dev/null 2>&1; echo "ncu k3 rc=$?"
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_prefill.py tests/test_gpu_parity.py -q -k "repeat_call or one_call_assign" > gpurun_out/memcheck_host_paths.txt 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/memcheck_host_paths.txt
