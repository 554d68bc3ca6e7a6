#!/bin/bash
# K3 instrumented variant next to the product library (PKV200_LIB=... to load):
#   phases  -DPKV_K3_PHASES (clock64 per softmax phase; PF_DEBUG=1 tools/bench_prefill.py prints them)
#   watchdog -DPKV_K3_WATCHDOG (mbarrier timeout trap)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2506_07311_b200/variants
for spec in "phases:PKV_K3_PHASES" "watchdog:PKV_K3_WATCHDOG" $EXTRA_VARIANTS; do
  name=${spec%%:*}; defs=${spec#*:}
  python - "$name" "$defs" <<'PY'
import sys
from paper_2506_07311_b200 import build as b
name, defs = sys.argv[1], sys.argv[2].split(",")
print(b.build(defines=defs, out=f"{b.PKG}/variants/lib_{name}.so", build_dir=f"{b.PKG}/build_{name}"))
PY
done
