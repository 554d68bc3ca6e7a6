"""A/B of the e2e decode step (pinned host in/out) with the output copied
back by a D2H (default) vs stored by the kernel straight into mapped pinned
memory (zero-copy), interleaved blocks in one process (diagnostic)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2506_07311_b200.batch as BM  # noqa: E402
from paper_2506_07311_b200.workloads import CONFIG_SHAPES, config_lengths  # noqa: E402

dev = torch.device("cuda:0")
lengths = config_lengths("c2")
hq, hkv, d, ps, _ = CONFIG_SHAPES["c2"]
pool, store, cfg = bench.build_cache(lengths, hq, hkv, d, ps, extra_tokens=1200, device=dev)
B = len(lengths)
batch = BM.DecodeBatch(store, list(range(B)), cfg)
q = torch.randn((B, hq, d)).bfloat16().pin_memory()
k = torch.randn((B, hkv, d)).bfloat16().pin_memory()
oh = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()
flush = torch.ones(64 << 20, device=dev)
res = {False: [], True: []}
for blk in range(20):
    zc = bool(blk % 2)
    BM._ZERO_COPY_OUT = zc
    for i in range(25):
        flush.sum()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        batch.step(q, k, k, out=oh)
        torch.cuda.current_stream().synchronize()
        if i >= 3:
            res[zc].append((time.perf_counter() - t0) * 1e6)
for zc, v in res.items():
    print("zero_copy" if zc else "d2h", "median %.1f us  p10 %.1f  p90 %.1f" % (np.median(v), np.percentile(v, 10), np.percentile(v, 90)))
