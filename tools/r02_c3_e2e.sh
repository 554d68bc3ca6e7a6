cd /root/repo
e2e() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], round(d['e2e']['ms_per_step']*1e3,1))"; }
B="--config c3 --context 8192 --batch 4 --no-cpu-baseline --no-prefill --no-check --steps 20 --warmup 5"
echo "default      $(timeout 200 python bench.py $B 2>/dev/null | e2e)"
echo "zc_kv=0      $(PKV_ZERO_COPY_KV=0 timeout 200 python bench.py $B 2>/dev/null | e2e)"
echo "zc_out=0     $(PKV_ZERO_COPY_OUT=0 timeout 200 python bench.py $B 2>/dev/null | e2e)"
echo "both=0       $(PKV_ZERO_COPY_KV=0 PKV_ZERO_COPY_OUT=0 timeout 200 python bench.py $B 2>/dev/null | e2e)"
echo "cluster=1    $(PKV_DECODE_CLUSTER=1 timeout 200 python bench.py $B 2>/dev/null | e2e)"
echo "b=64 2k      $(timeout 200 python bench.py --config c3 --context 2048 --batch 64 --no-cpu-baseline --no-prefill --no-check --steps 20 --warmup 5 2>/dev/null | e2e)"
echo "b=1 32k      $(timeout 200 python bench.py --config c3 --context 32768 --batch 1 --no-cpu-baseline --no-prefill --no-check --steps 20 --warmup 5 2>/dev/null | e2e)"
