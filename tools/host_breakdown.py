"""Per-call host cost (us) of the pieces of KvStore.assign and the prefill
paged_attention route, each call repeated in a tight loop (GPU box)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_07311_b200 import AttentionConfig, KvStore, MaskMeta, PagePool, _lib, paged_attention  # noqa: E402
from paper_2506_07311_b200 import attention as A  # noqa: E402
from paper_2506_07311_b200.store import _stream, to_device  # noqa: E402

dev = torch.device("cuda:0")
n, hq, hkv, d, ps = 8192, 32, 8, 128, 16
pool = PagePool(n // ps + 8, page_size=ps)
store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=dev)
pool.reserve(0, n)
k = torch.randn((n, hkv, d), device=dev).bfloat16()
pos = np.arange(n)
store.assign(0, pos, k, k)
cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
meta = MaskMeta.self_attention(store.batch_view([0]))
q = torch.randn((n, hq, d), device=dev).bfloat16()
lib = _lib.load()


def t(name, fn, reps=300):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    dt = (time.perf_counter() - t0) / reps * 1e6
    torch.cuda.synchronize()
    print(f"{name:44s} {dt:7.2f} us")


table = pool.table(0)
info, copies, cnt = store._assign_scratch(n)
mirror = pool.device_table(dev)
t("pool.table", lambda: pool.table(0))
t("np.asarray(pos, int64)", lambda: np.asarray(pos, dtype=np.int64))
t("_assign_scratch", lambda: store._assign_scratch(n))
t("pkv_pool_assign_prepare", lambda: lib.pkv_pool_assign_prepare(pool._h, table._handle, pos.ctypes.data, n,
                                                                  info.ctypes.data, copies.ctypes.data, copies.size,
                                                                  C.addressof(cnt)))
t("to_device(k)", lambda: to_device(k, dev, torch.bfloat16))
t("pool.device_table", lambda: pool.device_table(dev))
t("_stream", lambda: _stream(dev))
t("torch.cuda.current_device", torch.cuda.current_device)
t("table.logical_len", lambda: table.logical_len)
t("pkv_kv_append_range (launch)", lambda: lib.pkv_kv_append_range(
    k.data_ptr(), k.data_ptr(), n, int(info[4]), 0, mirror.data_ptr(), mirror.shape[1], ps, store._k_ptr,
    store._v_ptr, store.row_bytes, _stream(dev)), reps=100)
t("KvStore.assign total", lambda: store.assign(0, pos, k, k), reps=100)
print()
view = meta.view
rows = np.asarray([table.mirror_row], dtype=np.int32)
t("_check_queries", lambda: A._check_queries(q, meta, cfg))
t("pool.tables_info", lambda: pool.tables_info(view.ids))
t("pkv_prefill_supported", lambda: lib.pkv_prefill_supported(hq, hkv, d, ps, store.dtype_code))
t("_prefill_plan_meta", lambda: A._prefill_plan_meta(meta, cfg, rows, 1))
t("_prefill_route", lambda: A._prefill_route(meta, cfg, store.dtype_code, "prefill", rows))
route = A._prefill_route(meta, cfg, store.dtype_code, "prefill", rows)
t("_device_plan", lambda: A._device_plan(route, dev))
t("torch.empty out (134 MB)", lambda: torch.empty((n, hq, d), dtype=torch.float32, device=dev))
t("q.to(dtype).contiguous()", lambda: q.to(torch.bfloat16).contiguous())
dp = A._device_plan(route, dev)
out = torch.empty((n, hq, d), dtype=torch.float32, device=dev)


def mkargs():
    return _lib.PrefillArgs(
        q=q.data_ptr(), total_q=n, k_cache=store.k_cache.data_ptr(), v_cache=store.v_cache.data_ptr(),
        kv_dtype=store.dtype_code, cache_rows=store.k_cache.shape[0], block_table=mirror.data_ptr(),
        bt_stride=mirror.shape[1], page_size=ps, hq=hq, hkv=hkv, head_dim=d, scale=float(cfg.scale), causal=1,
        out=out.data_ptr(), out_dtype=_lib.PKV_F32, plan=dp.data_ptr(), n_items=route.n_items,
        prof_start=None, prof_stop=None)


t("PrefillArgs(...)", mkargs)
args = mkargs()
t("pkv_paged_prefill (launch)", lambda: lib.pkv_paged_prefill(C.byref(args), _stream(dev)), reps=30)
t("_launch_prefill", lambda: A._launch_prefill(q, meta, cfg, None, k=store.k_cache, v=store.v_cache,
                                               kv_code=store.dtype_code, bt=mirror, rows=rows,
                                               out_dtype=torch.float32, device=dev, route=route), reps=30)
t("paged_attention total", lambda: paged_attention(q, store, meta, cfg, precision="prefill"), reps=30)

# paged_attention's own body, section by section (prefill route)
from paper_2506_07311_b200.attention import _check_queries, _prefill_route, _q_tensor, _launch_prefill  # noqa: E402
acc = {}


def stamp(name, t0):
    t1 = time.perf_counter_ns()
    acc[name] = acc.get(name, 0) + (t1 - t0)
    return t1


def body():
    t0 = time.perf_counter_ns()
    _check_queries(q, meta, cfg)
    view = meta.view
    t0 = stamp("check", t0)
    n_pages, seq_row = store.pool.tables_info(view.ids)
    t0 = stamp("tables_info", t0)
    lengths = np.asarray(view.lengths, dtype=np.int64)
    bad = np.nonzero((lengths < 0) | (lengths > n_pages * store.page_size))[0]
    t0 = stamp("length check", t0)
    route = _prefill_route(meta, cfg, store.dtype_code, "prefill", seq_row)
    t0 = stamp("route", t0)
    qq, qcode = _q_tensor(q, dev)
    t0 = stamp("q_tensor", t0)
    mirror = store.pool.device_table(dev)
    t0 = stamp("device_table", t0)
    out = _launch_prefill(qq, meta, cfg, None, k=store.k_cache, v=store.v_cache, kv_code=store.dtype_code, bt=mirror,
                          rows=seq_row, out_dtype=torch.float32, device=dev, route=route)
    t0 = stamp("launch_prefill", t0)
    return out


for i in range(40):
    if i == 10:
        acc.clear()
    body()
torch.cuda.synchronize()
print({k: round(v / 30 / 1e3, 2) for k, v in acc.items()}, "sum", round(sum(acc.values()) / 30 / 1e3, 2))
acc.clear()
for i in range(40):
    if i == 10:
        acc.clear()
    torch.cuda.synchronize()
    body()
torch.cuda.synchronize()
print("isolated", {k: round(v / 30 / 1e3, 2) for k, v in acc.items()}, "sum", round(sum(acc.values()) / 30 / 1e3, 2))


def isolated(name, fn, reps=30):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    print(f"isolated {name:35s} p50 {np.median(ts):7.2f} us  min {np.min(ts):7.2f} us")


isolated("KvStore.assign", lambda: store.assign(0, pos, k, k))
isolated("paged_attention (prefill, repeat)", lambda: paged_attention(q, store, meta, cfg, precision="prefill"))
isolated("pkv_paged_prefill (launch only)", lambda: lib.pkv_paged_prefill(C.byref(args), _stream(dev)))
isolated("pkv_kv_append_range (launch only)", lambda: lib.pkv_kv_append_range(
    k.data_ptr(), k.data_ptr(), n, int(info[4]), 0, mirror.data_ptr(), mirror.shape[1], ps, store._k_ptr,
    store._v_ptr, store.row_bytes, _stream(dev)))
isolated("empty torch kernel (x.zero_())", lambda: out[:1].zero_())
