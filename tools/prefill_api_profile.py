"""Host time of one isolated paged_attention (prefill meta, 8192 tokens):
perf_counter around the call (no sync), with a cProfile of the same."""
import cProfile
import os
import pstats
import sys
import time

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
ts = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    paged_attention(q, store, meta, cfg)
    ts.append((time.perf_counter() - t0) * 1e6)
print("isolated paged_attention host us: p50 %.1f min %.1f" % (np.median(ts), np.min(ts)))
pr = cProfile.Profile()
for _ in range(20):
    torch.cuda.synchronize()
    pr.enable()
    paged_attention(q, store, meta, cfg)
    pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)

# piecewise host timing of one isolated call's steps
from paper_2506_07311_b200 import attention as A  # noqa: E402


def t(fn, reps=20):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        out.append((time.perf_counter() - t0) * 1e6)
    return round(float(np.median(out)), 1)


view = meta.view
rows = np.asarray([pool.table(0).mirror_row], dtype=np.int32)
route = A._prefill_route(meta, cfg, store.dtype_code, "auto", rows)
print({
    "check_queries": t(lambda: A._check_queries(q, meta, cfg)),
    "tables_info": t(lambda: pool.tables_info(view.ids)),
    "q_tensor": t(lambda: A._q_tensor(q, dev)),
    "prefill_route (native scan + memoised plan)": t(lambda: A._prefill_route(meta, cfg, store.dtype_code, "auto",
                                                                              rows)),
    "device_table": t(lambda: pool.device_table(dev)),
    "device_plan (generation hit)": t(lambda: A._device_plan(route, dev)),
    "launch_prefill_total": t(lambda: A._launch_prefill(q, meta, cfg, None, k=store.k_cache, v=store.v_cache,
                                                        kv_code=store.dtype_code, bt=pool.device_table(dev),
                                                        rows=rows, out_dtype=torch.float32, device=dev,
                                                        route=route)),
    "paged_attention_total": t(lambda: paged_attention(q, store, meta, cfg)),
})
