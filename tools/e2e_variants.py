"""C2 e2e step decomposed: where do the host/PCIe microseconds go?

Variants of DecodeBatch.step on the bench's C2 cache (all synchronous per
step, L2 flushed, median of 40):
  full      pinned host q/k/v in, pinned host out (the bench's e2e)
  dev_in    device-resident q/k/v, pinned host out
  dev_out   pinned host q/k/v in, device out
  dev_all   device in / device out (the API path without PCIe)
  host_only time until step() returns (no sync), full variant
Run with PKV_ZERO_COPY_IN=1 to read host q/k/v through mapped pointers."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_07311_b200.batch import DecodeBatch  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
_, lengths, hq, hkv, d, ps = bench.workload(cfgname, 0, 1)
pool, store, cfg = bench.build_cache(lengths, hq, hkv, d, ps, extra_tokens=2000, device=dev)
B = len(lengths)
batch = DecodeBatch(store, list(range(B)), cfg)
flush = bench.L2Flush(dev)
qh = torch.randn((B, hq, d)).bfloat16().pin_memory()
kh = torch.randn((B, hkv, d)).bfloat16().pin_memory()
vh = torch.randn((B, hkv, d)).bfloat16().pin_memory()
oh = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()
qd, kd, vd = qh.to(dev), kh.to(dev), vh.to(dev)
od = torch.empty((B, hq, d), dtype=torch.float32, device=dev)
st = torch.cuda.current_stream(dev)
res = {}
for name, (q, k, v, o) in {"full": (qh, kh, vh, oh), "dev_in": (qd, kd, vd, oh), "dev_out": (qh, kh, vh, od),
                           "dev_all": (qd, kd, vd, od)}.items():
    ts, th = [], []
    for i in range(50):
        flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        batch.step(q, k, v, out=o)
        t1 = time.perf_counter()
        st.synchronize()
        t2 = time.perf_counter()
        if i >= 10:
            ts.append((t2 - t0) * 1e6)
            th.append((t1 - t0) * 1e6)
    res[name] = (round(float(np.median(ts)), 1), round(float(np.median(th)), 1))
kv = sum(2 * (n + 100) * hkv * d * 2 for n in lengths)
print(cfgname, "zero_copy_in" if os.environ.get("PKV_ZERO_COPY_IN") == "1" else "h2d",
      {k: {"step_us": v[0], "host_return_us": v[1], "TB/s": round(kv / v[0] / 1e6, 2)} for k, v in res.items()})
