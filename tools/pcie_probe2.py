"""H2D latency distribution of the e2e step's input shapes (768 KiB as one
copy / three copies), synchronised per iteration like the e2e loop."""
import time
import numpy as np
import torch

dev = torch.device("cuda:0")
flushbuf = torch.ones(64 << 20, device=dev)
for label, sizes in (("1x768K", [768 << 10]), ("3x256K", [256 << 10] * 3), ("1x256K", [256 << 10]),
                     ("1x64K", [64 << 10]), ("1x4M", [4 << 20])):
    hs = [torch.empty(s, dtype=torch.uint8).pin_memory() for s in sizes]
    ds = [torch.empty(s, dtype=torch.uint8, device=dev) for s in sizes]
    ts = []
    for i in range(60):
        flushbuf.sum()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for h, d in zip(hs, ds):
            d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts = np.asarray(ts[10:])
    tot = sum(sizes)
    print(label, "us p10/p50/p90", np.percentile(ts, [10, 50, 90]).round(1), "GB/s p50", round(tot / np.median(ts) / 1e3, 1))
