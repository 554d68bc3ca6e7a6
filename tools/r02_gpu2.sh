#!/bin/bash
# probes: zero-copy host reads, K3 full ncu capture, small-batch decode times
timeout 120 ./tools/probes/zc_probe > gpurun_out/zc_probe.txt 2>&1
timeout 120 python tools/bench_prefill.py --iters 10 > gpurun_out/prefill.jsonl 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 3 -c 1 -o gpurun_out/prof_k3 -f python tools/bench_prefill.py --n 8192 --iters 1 > gpurun_out/p_k3.log 2>&1
timeout 400 bash tools/small_batch_auto.sh > gpurun_out/small_batch.txt 2>&1
cat gpurun_out/zc_probe.txt gpurun_out/prefill.jsonl gpurun_out/small_batch.txt
