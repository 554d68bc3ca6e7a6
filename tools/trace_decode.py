"""Per-CTA timeline of one tensor-core decode launch (debug)."""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2506_07311_b200 import _lib, MaskMeta, paged_attention
from paper_2506_07311_b200.batch import DecodeBatch

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
dev = torch.device('cuda', 0)
if B == 0:  # C2: MHA 32x128, 32 mixed lengths
    from oracle.workloads import config_lengths
    lens = config_lengths("c2")
    B = len(lens)
    pool, store, cfg = bench.build_cache(lens, 32, 32, 128, 16, 4, dev)
else:
    pool, store, cfg = bench.build_cache([ctx] * B, 32, 8, 128, 16, 4, dev)
meta = MaskMeta.decode(store.batch_view(list(range(B))))
q = torch.randn((B, 32, 128), device=dev).bfloat16()
ends = []
lib = _lib.load()
for _ in range(3):
    paged_attention(q, store, meta, cfg)
flush = torch.ones(64 << 20, device=dev)
flush.sum(); torch.cuda.synchronize()
print("trace on:", lib.pkv_debug_trace(1, None, 0), lib.pkv_last_error())
paged_attention(q, store, meta, cfg)
torch.cuda.synchronize()
buf = (C.c_uint64 * (148 * 64))()
print("trace read:", lib.pkv_debug_trace(-1, buf, 148 * 64), lib.pkv_last_error(), buf[0], buf[1], buf[63])
lib.pkv_debug_trace(0, None, 0)
t = np.array(buf, dtype=np.float64).reshape(148, 64)
t0 = t[:, 0][t[:, 0] > 0].min()
rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)
print("start spread (us): %.2f..%.2f" % (np.nanmin(rel[:, 0]), np.nanmax(rel[:, 0])))
print("plan done: median %.2f max %.2f" % (np.nanmedian(rel[:, 1]), np.nanmax(rel[:, 1])))
print("end: median %.2f max %.2f" % (np.nanmedian(rel[:, 63]), np.nanmax(rel[:, 63])))
busy = []
for b in range(148):
    tot = 0.0
    for k in range(20):
        s, c = rel[b, 2 + 3 * k], rel[b, 3 + 3 * k]
        if np.isnan(s):
            break
        tot += c - s
    busy.append(tot)
print("streaming time per CTA: mean %.1f min %.1f max %.1f; items per CTA: %s" % (
    np.mean(busy), np.min(busy), np.max(busy),
    np.bincount([sum(1 for k in range(20) if not np.isnan(rel[b, 2 + 3 * k])) for b in range(148)])))
ends = np.sort(rel[:, 63])
print("end-time deciles:", np.round(ends[::15], 1))
for b in [0, 1, 40, 100, 147]:
    items = []
    for k in range(20):
        s, c, m = rel[b, 2 + 3 * k], rel[b, 3 + 3 * k], rel[b, 4 + 3 * k]
        if np.isnan(s):
            break
        items.append("[%.1f chunks-done %.1f merged %.1f]" % (s, c, m))
    print("cta", b, "start %.1f plan %.1f" % (rel[b, 0], rel[b, 1]), " ".join(items), "end %.1f" % rel[b, 63])
