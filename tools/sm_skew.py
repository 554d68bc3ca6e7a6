"""Is the C2 end-time spread of K2-TC's CTAs systematic per SM?  Traces
several launches (pkv_debug_trace), records each CTA's SM and end time, and
reports the correlation of per-SM end times between launches and the
blockIdx -> SM mapping's stability."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_07311_b200 import MaskMeta, _lib, paged_attention  # noqa: E402
from paper_2506_07311_b200.workloads import config_lengths  # noqa: E402

dev = torch.device("cuda", 0)
lens = config_lengths("c2")
if os.environ.get("SHUFFLE"):  # the same sequences in another order: other work on every CTA
    lens = list(np.random.default_rng(int(os.environ["SHUFFLE"])).permutation(lens))
B = len(lens)
pool, store, cfg = bench.build_cache(lens, 32, 32, 128, 16, 4, dev)
meta = MaskMeta.decode(store.batch_view(list(range(B))))
q = torch.randn((B, cfg.head_count, 128), device=dev).bfloat16()
lib = _lib.load()
flush = torch.ones(64 << 20, device=dev)
for _ in range(3):
    paged_attention(q, store, meta, cfg)
runs = []
n = 256 * 8 * 32 + 256
for r in range(int(os.environ.get("RUNS", "6"))):
    flush.sum()
    torch.cuda.synchronize()
    lib.pkv_debug_trace(1, None, 0)
    paged_attention(q, store, meta, cfg)
    torch.cuda.synchronize()
    buf = (C.c_uint64 * n)()
    lib.pkv_debug_trace(-1, buf, n)
    lib.pkv_debug_trace(0, None, 0)
    arr = np.array(buf, dtype=np.float64)
    t = arr[:256 * 8 * 32].reshape(256, 8, 32)
    sm = arr[256 * 8 * 32:256 * 8 * 32 + 148].astype(int)
    tt = t[:148]
    t0 = tt[:, :, 0][tt[:, :, 0] > 0].min()
    rel = np.where(tt > 0, (tt - t0) / 1000.0, np.nan)
    ends = np.nanmax(rel[:, :, 31], axis=1)
    runs.append((sm, ends))
sm0 = runs[0][0]
print("blockIdx->SM identical across runs:", [bool(np.array_equal(sm0, s)) for s, _ in runs])
per_sm = []
for s, e in runs:
    v = np.full(148, np.nan)
    v[s] = e
    per_sm.append(v)
per_sm = np.array(per_sm)
per_cta = np.array([e for _, e in runs])
print("end spread per run (min/median/max us):", [(round(np.nanmin(e), 1), round(np.nanmedian(e), 1),
                                                    round(np.nanmax(e), 1)) for e in per_cta])
def corr(m):
    c = np.corrcoef(m)
    return round(float(np.mean(c[np.triu_indices(len(m), 1)])), 3)
print("mean pairwise corr of end times by SM:", corr(per_sm), " by CTA:", corr(per_cta))
mean_sm = np.nanmean(per_sm, 0)
order = np.argsort(mean_sm)
print("slowest SMs (mean end us):", [(int(i), round(float(mean_sm[i]), 1)) for i in order[-12:]])
print("fastest SMs:", [(int(i), round(float(mean_sm[i]), 1)) for i in order[:12]])
# GPC-ish structure: SM id // 2 = TPC
tpc = np.arange(148) // 2
print("per-TPC-pair-of-SMs end corr within TPC:", round(float(np.corrcoef(mean_sm[0::2], mean_sm[1::2])[0, 1]), 3))
tag = os.environ.get("SHUFFLE", "0")
sys.path.insert(0, "tests")
from test_decode_plan import parse  # noqa: E402
lens_now = [int(x) for x in meta.view.lengths]
rows_now = [int(pool.table(b).mirror_row) for b in range(B)]
P = parse(_lib.attention_plan(np.asarray(lens_now, np.int32), np.asarray(rows_now, np.int32), 16,
                              cfg.head_count, cfg.kv_head_count))
cta, items = P["cta"], P["items"]
pages = np.array([sum(r[3] - r[2] for r in items[cta[c]:cta[c + 1]]) for c in range(148)], dtype=np.float64)
cuts = np.array([sum(1 for r in items[cta[c]:cta[c + 1]] if r[4] >= 0) for c in range(148)])
nit = np.array([cta[c + 1] - cta[c] for c in range(148)])
me = per_cta.mean(0)
print("corr(end, pages) %.3f  corr(end, items) %.3f  corr(end, cuts) %.3f" % (
    np.corrcoef(me, pages)[0, 1], np.corrcoef(me, nit)[0, 1], np.corrcoef(me, cuts)[0, 1]))
print("pages per CTA min/median/max:", pages.min(), np.median(pages), pages.max())
print("per-SM mean end (us), SM id order, 16 per row:")
for r0 in range(0, 148, 16):
    print("  sm %3d:" % r0, " ".join("%5.1f" % x for x in mean_sm[r0:r0 + 16]))
print("per-SM end rate (us per 100 pages), SM id order:")
rate = np.full(148, np.nan)
rate[sm0] = me / pages * 100
for r0 in range(0, 148, 16):
    print("  sm %3d:" % r0, " ".join("%5.2f" % x for x in rate[r0:r0 + 16]))

np.save(f"gpurun_out/sm_skew_{tag}.npy", np.stack([mean_sm, rate]))
