cd /root/repo
for pt in 1:2048 1:8192 2:8192 4:8192; do
  b=${pt%%:*}; c=${pt##*:}
  for cl in 0 16 8 4; do
    v=$(PKV_DECODE_CLUSTER=$cl timeout 120 python bench.py --config c3 --context $c --batch $b --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-prefill --no-check 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1))")
    echo "b=$b ctx=$c cluster=$cl ${v}us"
  done
done
