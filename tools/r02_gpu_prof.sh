#!/bin/bash
# round-2 evidence: full GPU suite, ncu --set full of K2-TC (C2, C3 8k x64, C5, C2 fragmented) and K3, launch list
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
K="--set full --clock-control none --import-source on -k regex:decode_tc -s 2 -c 1 -f"
timeout 400 ncu $K -o gpurun_out/r02_k2_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill --no-c5 --no-check > /dev/null 2>&1
timeout 400 ncu $K -o gpurun_out/r02_k2_c2frag python bench.py --fragment --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill --no-c5 --no-check > /dev/null 2>&1
timeout 400 ncu $K -o gpurun_out/r02_k2_c3 python bench.py --config c3 --context 8192 --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill --no-check > /dev/null 2>&1
timeout 600 ncu $K -o gpurun_out/r02_k2_c5 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill --no-check > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 3 -c 1 -f -o gpurun_out/r02_k3 python tools/bench_prefill.py --n 8192 --iters 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill --no-c5 > /dev/null 2>&1
ls -la gpurun_out | grep r02
