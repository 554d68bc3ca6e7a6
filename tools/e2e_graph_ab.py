"""C2 e2e step with and without the CUDA-graph step (same cache, same
buffers): per-step wall time, graph launches / builds."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_07311_b200.batch import DecodeBatch  # noqa: E402

dev = torch.device("cuda:0")
_, lengths, hq, hkv, d, ps = bench.workload("c2", 0, 1)
pool, store, cfg = bench.build_cache(lengths, hq, hkv, d, ps, extra_tokens=1200, device=dev)
B = len(lengths)
flush = bench.L2Flush(dev)
host = [tuple(torch.randn(s).bfloat16().pin_memory() for s in ((B, hq, d), (B, hkv, d), (B, hkv, d)))
        for _ in range(4)]
oh = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()
st = torch.cuda.current_stream(dev)
dev_in = len(sys.argv) > 1 and sys.argv[1] == "dev"
if dev_in:  # a model's layer: q / k / v produced on the device, output kept there
    host = [tuple(t.to(dev) for t in h) for h in host]
    oh = torch.empty((B, hq, d), dtype=torch.float32, device=dev)
for mode in (False, True, False, True):
    batch = DecodeBatch(store, list(range(B)), cfg)
    batch.use_graph = mode
    ts = []
    for i in range(60):
        q, k, v = host[i % 4]
        flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        batch.step(q, k, v, out=oh)
        t1 = time.perf_counter()
        st.synchronize()
        t2 = time.perf_counter()
        if i >= 10:
            ts.append(((t2 - t0) * 1e6, (t1 - t0) * 1e6))
    ts = np.asarray(ts)
    print("graph" if mode else "plain", "step p50 %.1f us  host-return p50 %.1f us" % tuple(np.median(ts, 0)),
          "stats", batch.graph_stats())
