"""Per-warp timeline of one tensor-core decode launch (debug).

    python tools/trace_decode.py B CTX     # C3 GQA shape, B sequences of CTX
    python tools/trace_decode.py 0         # C2 (MHA 32x128, 32 mixed lengths)
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2506_07311_b200 import MaskMeta, _lib, paged_attention  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
dev = torch.device('cuda', 0)
if B == 0:
    from paper_2506_07311_b200.workloads import config_lengths
    lens = config_lengths("c2")
    B = len(lens)
    pool, store, cfg = bench.build_cache(lens, 32, 32, 128, 16, 4, dev)
else:
    pool, store, cfg = bench.build_cache([ctx] * B, 32, 8, 128, 16, 4, dev)
meta = MaskMeta.decode(store.batch_view(list(range(B))))
q = torch.randn((B, cfg.head_count, 128), device=dev).bfloat16()
lib = _lib.load()
for _ in range(3):
    paged_attention(q, store, meta, cfg)
import os
flush = torch.ones(64 << 20, device=dev)
if not os.environ.get("WARM"):
    flush.sum()
torch.cuda.synchronize()
# event time of the same launch (cold L2), for comparison with the in-kernel span
ev = []
for _ in range(10):
    flush.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    paged_attention(q, store, meta, cfg)
    e1.record()
    torch.cuda.synchronize()
    ev.append(e0.elapsed_time(e1) * 1e3)
print("event-timed paged_attention (us): median %.1f min %.1f" % (np.median(ev), np.min(ev)))
flush.sum()
torch.cuda.synchronize()
lib.pkv_debug_trace(1, None, 0)
paged_attention(q, store, meta, cfg)
torch.cuda.synchronize()
n = 256 * 8 * 32
buf = (C.c_uint64 * n)()
lib.pkv_debug_trace(-1, buf, n)
lib.pkv_debug_trace(0, None, 0)
t = np.array(buf, dtype=np.float64).reshape(256, 8, 32)[:148]
t0 = t[:, :, 0][t[:, :, 0] > 0].min()
rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)
print("kernel span (us): %.1f   plan done median %.2f" % (np.nanmax(rel[:, :, 31]), np.nanmedian(rel[:, :, 1])))
print("prologue medians: start_item %.2f  first issue %.2f  prologue issued %.2f  | merge: stored %.2f  "
      "cluster_wait %.2f  pushed %.2f  end %.2f" % tuple(np.nanmedian(rel[:, :, s]) for s in (24, 25, 26, 5, 27, 28, 31)))
gaps = {"start->first data": [], "first data->chunks done": [], "chunks done->stored": [],
        "stored->next start": []}
for c in range(148):
    for w in range(8):
        for k in range(7):
            s, f, d, st = rel[c, w, 2 + 4 * k: 6 + 4 * k]
            if np.isnan(s):
                break
            if not np.isnan(f):
                gaps["start->first data"].append(f - s)
                gaps["first data->chunks done"].append(d - f)
            gaps["chunks done->stored"].append(st - d)
            nxt = rel[c, w, 2 + 4 * (k + 1)] if k < 6 else np.nan
            if not np.isnan(nxt):
                gaps["stored->next start"].append(nxt - st)
for k_, v in gaps.items():
    v = np.array(v)
    if v.size == 0:
        continue
    print("%-26s n=%5d mean %6.2f  p50 %6.2f  p90 %6.2f  max %6.2f  sum/warp %6.2f" % (
        k_, v.size, v.mean(), np.median(v), np.percentile(v, 90), v.max(), v.sum() / (148 * 8)))
ends = np.nanmax(rel[:, :, 31], axis=1)
starts = np.nanmin(rel[:, :, 0], axis=1)
print("CTA start deciles:", np.round(np.sort(starts)[::15], 1))
first = np.nanmin(rel[:, :, 2], axis=1)
print("CTA first-item deciles:", np.round(np.sort(first)[::15], 1))
print("CTA end deciles:", np.round(np.sort(ends)[::15], 1))
for c in [0, int(np.argsort(ends)[len(ends) // 2]), int(np.nanargmax(ends))]:
    print("cta", c)
    for w in range(8):
        items = []
        for k in range(7):
            s, f, d, st = rel[c, w, 2 + 4 * k: 6 + 4 * k]
            if np.isnan(s):
                break
            items.append("[%.1f f%.1f d%.1f s%.1f]" % (s, f, d, st))
        print("  w%d" % w, " ".join(items), "merged %.1f stored %.1f finished %.1f end %.1f" % (
            rel[c, w, 28], rel[c, w, 29], rel[c, w, 30], rel[c, w, 31]))

# per-CTA correlation with the plan: items, pages, cut pieces
if os.environ.get("CORR"):
    sys.path.insert(0, "tests")
    from test_decode_plan import parse
    lens_now = [int(x) for x in meta.view.lengths]
    rows_now = [int(pool.table(b).mirror_row) for b in range(B)]
    P = parse(_lib.attention_plan(np.asarray(lens_now, np.int32), np.asarray(rows_now, np.int32), 16,
                                  cfg.head_count, cfg.kv_head_count))
    cta, items = P["cta"], P["items"]
    recs = []
    for c in range(min(148, P["grid"])):
        its = items[cta[c]:cta[c + 1]]
        pages = int(sum(r[3] - r[2] for r in its))
        cuts = int(sum(1 for r in its if r[4] >= 0))
        recs.append((ends[c], c, len(its), pages, cuts))
    recs.sort()
    print("fastest:", [(round(e, 1), c, n, p, k) for e, c, n, p, k in recs[:6]])
    print("slowest:", [(round(e, 1), c, n, p, k) for e, c, n, p, k in recs[-10:]])
    import collections
    by_items = collections.defaultdict(list)
    for e, c, n, p, k in recs:
        by_items[n].append(e)
    print("end time by item count:", {n: round(float(np.mean(v)), 1) for n, v in sorted(by_items.items())})
    by_cuts = collections.defaultdict(list)
    for e, c, n, p, k in recs:
        by_cuts[k].append(e)
    print("end time by cut pieces:", {n: round(float(np.mean(v)), 1) for n, v in sorted(by_cuts.items())})
    # epilogue (chunks done -> stored) and streaming time per item, cut vs whole
    ep = {"whole": [], "cut": []}
    st_rate = {"whole": [], "cut": []}
    for c in range(min(148, P["grid"])):
        its = items[cta[c]:cta[c + 1]]
        for k, r in enumerate(its[:7]):
            kind = "cut" if r[4] >= 0 else "whole"
            for w in range(8):
                s_, f_, d_, st_ = rel[c, w, 2 + 4 * k: 6 + 4 * k]
                if not np.isnan(d_) and not np.isnan(st_):
                    ep[kind].append(st_ - d_)
                if not np.isnan(f_) and not np.isnan(d_) and r[3] > r[2]:
                    st_rate[kind].append((d_ - f_) / (r[3] - r[2]))
    for kind in ep:
        if ep[kind]:
            print("%-5s items: epilogue us p50 %.2f mean %.2f | stream us/page p50 %.3f" % (
                kind, np.median(ep[kind]), np.mean(ep[kind]), np.median(st_rate[kind]) if st_rate[kind] else -1))
