"""Continuous-batching serving simulation on the device engine (SURVEY.md §8
f-3: workload traces driving real GPU pools, plus the memory audit).

Seeded requests arrive (prompt log-uniform in [128, 8192], generation length
uniform in [16, 256]); every step admits the arrivals — reserve, K1 append of
the prompt, K3 causal prefill over it — then advances every live request by
one token with a single fused append+decode launch (DecodeBatch), and frees
the finished ones (their pages go back on the LIFO free stack, so later
requests get scattered tables).  One attention layer, Llama-3-8B GQA shape,
bf16, page 16.  Reports decode / prefill throughput and the KV overhead
(reference workload.account: charged slots / minimum - 1) at the peak.

    python tools/serve_sim.py [--requests 256] [--rate 4] [--seed 0]
"""

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_07311_b200 import AttentionConfig, KvStore, MaskMeta, PagePool, paged_attention  # noqa: E402
from paper_2506_07311_b200.batch import DecodeBatch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=256)
    ap.add_argument("--rate", type=float, default=4.0, help="mean arrivals per decode step")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--pool-pages", type=int, default=1 << 17)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    hq, hkv, d, ps = 32, 8, 128, 16
    rng = np.random.default_rng(args.seed)
    prompts = np.exp(rng.uniform(math.log(128), math.log(8192), args.requests)).astype(int)
    gens = rng.integers(16, 257, args.requests)
    arrivals = np.cumsum(rng.exponential(1.0 / args.rate, args.requests)).astype(int)
    pool = PagePool(args.pool_pages, page_size=ps)
    store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=dev)
    cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
    batch = None
    live = {}  # request -> tokens still to generate
    nxt = 0
    step = 0
    stats = {"decode_tokens": 0, "prefill_tokens": 0, "decode_ms": 0.0, "prefill_ms": 0.0, "steps": 0,
             "peak_live": 0, "peak_overhead": 0.0, "peak_tokens": 0, "peak_pages": 0}
    g = torch.Generator(device=dev).manual_seed(args.seed)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t_wall = time.perf_counter()
    while nxt < args.requests or live:
        # admissions: prompt append (K1) + causal prefill (K3)
        admitted = []
        while nxt < args.requests and arrivals[nxt] <= step:
            n = int(prompts[nxt])
            pool.reserve(nxt, n)
            k = torch.randn((n, hkv, d), generator=g, device=dev).bfloat16()
            q = torch.randn((n, hq, d), generator=g, device=dev).bfloat16()
            e0, e1 = ev(), ev()
            e0.record()
            store.assign(nxt, np.arange(n), k, k)
            paged_attention(q, store, MaskMeta.self_attention(store.batch_view([nxt])), cfg)
            e1.record()
            admitted.append((e0, e1))
            live[nxt] = int(gens[nxt])
            stats["prefill_tokens"] += n
            nxt += 1
        if not live:
            step += 1
            continue
        ids = sorted(live)
        if batch is None:
            batch = DecodeBatch(store, ids, cfg, capacity=64)
        else:
            batch.set_sequences(ids)
        B = len(ids)
        q = torch.randn((B, hq, d), generator=g, device=dev).bfloat16()
        kn = torch.randn((B, hkv, d), generator=g, device=dev).bfloat16()
        e0, e1 = ev(), ev()
        e0.record()
        batch.step(q, kn, kn)
        e1.record()
        torch.cuda.synchronize()
        stats["decode_ms"] += e0.elapsed_time(e1)
        stats["prefill_ms"] += sum(a.elapsed_time(b) for a, b in admitted)
        stats["decode_tokens"] += B
        stats["steps"] += 1
        # memory audit at this step (reference workload.account definition)
        lens = np.asarray([pool.table(r).logical_len for r in ids], dtype=np.int64)
        tokens = int(lens.sum())
        charged = int((-(-lens // ps)).sum()) * ps
        if tokens > stats["peak_tokens"]:
            stats.update(peak_tokens=tokens, peak_overhead=charged / tokens - 1.0, peak_live=B,
                         peak_pages=pool.census().live_pages)
        for r in ids:
            live[r] -= 1
            if live[r] == 0:
                del live[r]
                pool.free(r)
        step += 1
    wall = time.perf_counter() - t_wall
    census = pool.census()
    print(json.dumps({
        "workload": f"{args.requests} requests, prompts 128-8192 (log-uniform), 16-256 generated tokens, "
                    f"~{args.rate}/step arrivals, GQA 32q/8kv x128 bf16, page {ps}, one attention layer",
        "steps": stats["steps"], "decode_tokens": stats["decode_tokens"], "prefill_tokens": stats["prefill_tokens"],
        "decode_tok_per_s_device": round(stats["decode_tokens"] / (stats["decode_ms"] * 1e-3), 1),
        "prefill_tok_per_s_device": round(stats["prefill_tokens"] / (stats["prefill_ms"] * 1e-3), 1),
        "mean_decode_step_us": round(1e3 * stats["decode_ms"] / stats["steps"], 1),
        "peak_live_sequences": stats["peak_live"], "peak_tokens": stats["peak_tokens"],
        "kv_overhead_at_peak": round(stats["peak_overhead"], 5), "peak_live_pages": stats["peak_pages"],
        "pool_after": {"live": census.live_pages, "free": census.free_pages, "never": census.never_allocated},
        "wall_s": round(wall, 2)}))


if __name__ == "__main__":
    main()
