#!/bin/bash
# closing pass: GPU suite, smoke, bench line + C3 sweep (JSON lines on stderr), reference arm, launch list, ncu of K2-TC on C2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1500 python bench.py --sweep > gpurun_out/bench_main.json 2> gpurun_out/bench_sweep.err; echo "bench rc=$?"
grep '^{' gpurun_out/bench_sweep.err > gpurun_out/c3_sweep.jsonl; wc -l gpurun_out/c3_sweep.jsonl
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
K="--set full --clock-control none --import-source on -k regex:decode_tc -s 2 -c 1 -f"
timeout 400 ncu $K -o gpurun_out/r02_k2_c2_final python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill --no-c5 --no-check > /dev/null 2>&1; echo "ncu k2 rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_main.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step", "gpu_launches", "parity_checked")}, d["clocks"])
print("roofline", {k: d["roofline"][k] for k in ("achieved", "frac", "frac_of_read_probe")})
print("e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], "c5", d["c5"]["value"])
print("c4", {k: d["prefill_c4"][k] for k in ("kernel_ms", "tflops", "api_ms", "api_pipelined_ms", "append_ms", "append_gbs")})
r = json.loads(open("gpurun_out/bench_ref.json").read().strip().splitlines()[-1])
print("ref", r.get("value"), r.get("unit"), r.get("cpu_baseline", {}).get("cores"))
PY
