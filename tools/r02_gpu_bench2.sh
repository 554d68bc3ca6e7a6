#!/bin/bash
# default bench (C2 + C5 + C4 + e2e), fragmented-pool bench, C3 sweep with clocks
timeout 600 python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err
timeout 600 python bench.py --fragment --no-cpu-baseline --no-prefill > gpurun_out/bench_frag.json 2> gpurun_out/bench_frag.err
timeout 1500 python bench.py --sweep --no-cpu-baseline --no-e2e --no-prefill --no-c5 --steps 5 --warmup 3 > /dev/null 2> gpurun_out/sweep.err
grep "^SWEEP" gpurun_out/sweep.err | sed 's/^SWEEP //' > gpurun_out/c3_sweep.jsonl
wc -l gpurun_out/c3_sweep.jsonl
cat gpurun_out/bench_main.json | head -c 3000
