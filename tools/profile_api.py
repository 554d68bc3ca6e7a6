"""cProfile of the host side of paged_attention (prefill and decode metas)."""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_07311_b200 import AttentionConfig, KvStore, MaskMeta, PagePool, paged_attention  # noqa: E402

dev = torch.device("cuda:0")
n, hq, hkv, d, ps = 8192, 32, 8, 128, 16
pool = PagePool(n // ps + 8, page_size=ps)
store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=dev)
pool.reserve(0, n)
k = torch.randn((n, hkv, d), device=dev).bfloat16()
store.assign(0, np.arange(n), k, k)
cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
meta = MaskMeta.self_attention(store.batch_view([0]))
q = torch.randn((n, hq, d), device=dev).bfloat16()
for _ in range(3):
    paged_attention(q, store, meta, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    paged_attention(q, store, meta, cfg)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

# KvStore.assign of the whole prompt (K1): host side
pos = np.arange(n)
for _ in range(3):
    store.assign(0, pos, k, k)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    store.assign(0, pos, k, k)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
