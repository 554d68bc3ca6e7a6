#!/bin/bash
# e2e decomposition: H2D copies vs zero-copy inputs
timeout 300 python tools/e2e_variants.py c2 > gpurun_out/e2e_var.txt 2>&1
PKV_ZERO_COPY_IN=1 timeout 300 python tools/e2e_variants.py c2 >> gpurun_out/e2e_var.txt 2>&1
timeout 120 python tools/pcie_probe2.py >> gpurun_out/e2e_var.txt 2>&1
cat gpurun_out/e2e_var.txt
