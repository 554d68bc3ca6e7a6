# full ncu captures of the dominant kernels + the bench launch list (1 GPU)
set -x
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 2 -c 1 -o gpurun_out/prof_k2_c2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_k2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 2 -c 1 -o gpurun_out/prof_k2_c3 -f python bench.py --config c3 --context 8192 --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_k2c3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 3 -c 1 -o gpurun_out/prof_k3 -f python tools/bench_prefill.py --n 8192 --iters 1 > gpurun_out/p_k3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > /dev/null 2>&1
ls -la gpurun_out
