import os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2506_07311_b200.batch import DecodeBatch
from paper_2506_07311_b200.workloads import CONFIG_SHAPES, config_lengths
dev = torch.device("cuda:0")
lengths = config_lengths("c2")
hq, hkv, d, ps, _ = CONFIG_SHAPES["c2"]
pool, store, cfg = bench.build_cache(lengths, hq, hkv, d, ps, extra_tokens=200, device=dev)
B = len(lengths)
batch = DecodeBatch(store, list(range(B)), cfg)
q = torch.randn((B, hq, d)).bfloat16().pin_memory()
k = torch.randn((B, hkv, d)).bfloat16().pin_memory()
oh = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()
ph = {"h2d_issue": [], "step_host": [], "d2h_issue": [], "sync": [], "total": []}
for i in range(60):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    qd = q.to(dev, non_blocking=True); kd = k.to(dev, non_blocking=True); vd = k.to(dev, non_blocking=True)
    t1 = time.perf_counter()
    o = batch.step(qd, kd, vd)
    t2 = time.perf_counter()
    oh.copy_(o, non_blocking=True)
    t3 = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    t4 = time.perf_counter()
    if i >= 10:
        for kk, v in zip(ph, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
            ph[kk].append(v * 1e6)
print({kk: round(float(np.median(v)), 1) for kk, v in ph.items()})

# split step(): prepare() (allocator + metadata + plan + page clears) vs the launch half
import ctypes as C
from paper_2506_07311_b200 import _lib
ph2 = {"prepare": [], "launch_half": [], "native_prepare_only": []}
lib = _lib.load()
for i in range(60):
    torch.cuda.synchronize()
    qd = q.to(dev, non_blocking=True); kd = k.to(dev, non_blocking=True); vd = k.to(dev, non_blocking=True)
    t0 = time.perf_counter()
    batch.prepare()
    t1 = time.perf_counter()
    o = batch.step(qd, kd, vd, advance=False)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    if i >= 10:
        ph2["prepare"].append((t1 - t0) * 1e6)
        ph2["launch_half"].append((t2 - t1) * 1e6)
print({kk: round(float(np.median(v)), 1) for kk, v in ph2.items() if v})
t0 = time.perf_counter()
for i in range(200):
    pool.device_table(dev)
print("device_table us", (time.perf_counter() - t0) / 200 * 1e6)
t0 = time.perf_counter()
for i in range(200):
    torch.empty((B, hq, d), dtype=torch.float32, device=dev)
print("torch.empty us", (time.perf_counter() - t0) / 200 * 1e6)
t0 = time.perf_counter()
for i in range(200):
    torch.cuda.current_stream(dev)
print("current_stream us", (time.perf_counter() - t0) / 200 * 1e6)
