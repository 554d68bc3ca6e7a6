# K3 bring-up: parity tests, then timing (each bounded)
timeout 300 python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -30 > gpurun_out/k3_pytest.log
timeout 200 python tools/bench_prefill.py > gpurun_out/k3_bench.log 2>&1
cat gpurun_out/k3_pytest.log gpurun_out/k3_bench.log
