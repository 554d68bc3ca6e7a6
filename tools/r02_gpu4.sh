#!/bin/bash
# fast-path step test + e2e variants: H2D vs zero-copy inputs x L2 prefetch of the segment head
timeout 600 python -m pytest tests/test_gpu_decode_tc.py -x -q -k "fast_path or host_buffer" > gpurun_out/t4.log 2>&1; tail -2 gpurun_out/t4.log
timeout 60 python tools/pcie_probe2.py 2>&1 | head -2
for zc in 0 1; do for pf in 0 8 24; do
  echo "== zc=$zc prefetch=$pf"
  PKV_ZERO_COPY_IN=$zc PKV_DECODE_L2_PREFETCH=$pf timeout 300 python tools/e2e_variants.py c2 2>&1 | head -2
done; done
