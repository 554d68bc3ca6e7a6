#!/bin/bash
# A/B of two library builds on the C3 small-batch points (same box, interleaved)
# usage: tools/ab_c3.sh OLD.so NEW.so "1:2048 1:32768 8:2048"
OLD=$1; NEW=$2; PTS=${3:-"1:2048 1:8192 1:32768 4:8192 8:2048 8:32768"}
for pt in $PTS; do
  b=${pt%%:*}; c=${pt##*:}
  for rep in 1 2; do
    for lib in "$OLD" "$NEW"; do
      v=$(PKV200_LIB=$lib python bench.py --config c3 --context $c --batch $b --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-prefill 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1))")
      echo "b=$b ctx=$c $(basename $lib) ${v}us"
    done
  done
done
