"""Host<->device copy bandwidth on the box, with the process bound to the
GPU-local CPUs (NVML affinity) or not: the e2e step's PCIe legs."""
import os
import sys
import time

import numpy as np
import torch


def probe(tag):
    dev = torch.device("cuda:0")
    res = {}
    for nbytes in (256 << 10, 768 << 10, 8 << 20, 64 << 20):
        h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        for direction in ("h2d", "d2h"):
            ts = []
            for i in range(30):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if direction == "h2d":
                    d.copy_(h, non_blocking=True)
                else:
                    h.copy_(d, non_blocking=True)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts[5:]))
            res[f"{direction}_{nbytes >> 10}KiB"] = f"{ms * 1e3:.1f}us {nbytes / ms / 1e6:.1f}GB/s"
    print(tag, res, flush=True)


print("cpus", len(os.sched_getaffinity(0)), "numa nodes", sorted(os.listdir("/sys/devices/system/node")) if os.path.isdir("/sys/devices/system/node") else None)
probe("default")
try:
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    ncpu = os.cpu_count()
    words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
    cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if m >> b & 1]
    print("gpu-local cpus", len(cpus), cpus[:8], "...")
    os.sched_setaffinity(0, cpus)
    probe("gpu_local")
except Exception as e:
    print("affinity failed", e)
