set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/r1_bench.log 2>&1
timeout 300 bash tools/sweep.sh > gpurun_out/r1_sweep.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r1_ncu_bench.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:decode -s 6 -c 2 -o gpurun_out/r1_k2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r1_ncu_full.log 2>&1
tail -3 gpurun_out/*.log
