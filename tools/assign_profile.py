"""KvStore.assign of one 8192-token prompt: host time of the call (no sync)
vs the K1 kernel's device time, and a line profile of the host side."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_07311_b200 import KvStore, PagePool  # noqa: E402

dev = torch.device("cuda:0")
n, hkv, d, ps = 8192, 8, 128, 16
pool = PagePool(n // ps + 8, page_size=ps)
store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=dev)
pool.reserve(0, n)
k = torch.randn((n, hkv, d), device=dev).bfloat16()
pos = np.arange(n)
for _ in range(5):
    store.assign(0, pos, k, k)
torch.cuda.synchronize()
host, dev_t = [], []
for _ in range(20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    store.assign(0, pos, k, k)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    host.append((t1 - t0) * 1e6)
    dev_t.append(e0.elapsed_time(e1) * 1e3)
print("assign host us p50 %.1f  event us p50 %.1f" % (np.median(host), np.median(dev_t)))
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    store.assign(0, pos, k, k)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
