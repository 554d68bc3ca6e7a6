set -x
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5.log 2>&1
tail -1 gpurun_out/c5.log | cut -c1-1500
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_decode_tc.py -x -q -k "fused_append or general_meta" > gpurun_out/memcheck_k2.log 2>&1; echo "memcheck k2 rc=$?"; tail -3 gpurun_out/memcheck_k2.log
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_prefill.py -x -q -k "suffix or fp16 or bitwise" > gpurun_out/memcheck_k3.log 2>&1; echo "memcheck k3 rc=$?"; tail -3 gpurun_out/memcheck_k3.log
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_decode_tc.py -x -q -k "general_meta" > gpurun_out/racecheck_k2.log 2>&1; echo "racecheck k2 rc=$?"; tail -3 gpurun_out/racecheck_k2.log
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/memcheck_parity.log 2>&1; echo "memcheck parity rc=$?"; tail -3 gpurun_out/memcheck_parity.log
