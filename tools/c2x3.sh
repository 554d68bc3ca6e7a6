cd /root/repo
for rep in 1 2 3; do timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-prefill --no-c5 --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'])"; done
