"""Prefix sharing (SPEC AC6): fork N children off one long
prompt and decode them together.

* fork: host allocator fork (O(1) in the prefix: pages are shared by
  refcount) + one batched K0b copy of the partial last page;
* memory: live pages with sharing vs N private copies;
* decode: one DecodeBatch step over the N children (K1 fused into K2-TC);
  every child attends over the shared prefix pages, so the logical KV bytes
  read exceed what HBM delivers (L2 reuse across children).
Prints one JSON line.
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_07311_b200 import AttentionConfig, KvStore, PagePool  # noqa: E402
from paper_2506_07311_b200.batch import DecodeBatch  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    n_prefix, children, steps = int(os.environ.get("PREFIX", 8190)), int(os.environ.get("CHILDREN", 64)), 8
    hq, hkv, d, ps = 32, 8, 128, 16
    pool = PagePool(n_prefix // ps + children * (2 + steps // ps + 1) + 16, ps)
    store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=dev)
    cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
    pool.reserve("parent", n_prefix)
    k = torch.randn((n_prefix, hkv, d), device=dev).bfloat16()
    store.assign("parent", np.arange(n_prefix), k, k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for c in range(children):
        pool.fork("parent", c, n_prefix)
    torch.cuda.synchronize()
    fork_us = (time.perf_counter() - t0) * 1e6 / children
    census = pool.census()
    private_pages = children * -(-n_prefix // ps)
    batch = DecodeBatch(store, list(range(children)), cfg)
    q = torch.randn((children, hq, d), device=dev).bfloat16()
    kn = torch.randn((children, hkv, d), device=dev).bfloat16()
    for _ in range(2):
        batch.step(q, kn, kn)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s, e in ev:
        s.record()
        batch.step(q, kn, kn)
        e.record()
    torch.cuda.synchronize()
    ms = float(np.median([s.elapsed_time(e) for s, e in ev]))
    ctx = n_prefix + 2 + steps // 2
    logical = children * ctx * hkv * d * 2 * 2
    unique = (ctx + children * (2 + steps)) * hkv * d * 2 * 2
    print(json.dumps({
        "workload": f"{children} children forked off a {n_prefix}-token prompt, GQA 32q/8kv x128 bf16, page {ps}",
        "fork_us_per_child": round(fork_us, 1), "live_pages": census.live_pages,
        "pages_without_sharing": private_pages + children, "memory_saving": round(1 - census.live_pages / (private_pages + children), 4),
        "decode_step_ms": ms, "logical_kv_gb_per_s": round(logical / (ms * 1e-3) / 1e9, 1),
        "unique_kv_gb_per_s": round(unique / (ms * 1e-3) / 1e9, 1),
        "tokens_per_s": round(children / (ms * 1e-3), 1)}))


if __name__ == "__main__":
    main()
