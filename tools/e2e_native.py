"""Host-side cost breakdown of the one-call decode step (pkv_decode_step)
on C2: DecodeBatch.step with pinned host q/k/v/out (diagnostic)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_07311_b200 import _lib  # noqa: E402
from paper_2506_07311_b200.batch import DecodeBatch  # noqa: E402
from paper_2506_07311_b200.store import _stream  # noqa: E402
from paper_2506_07311_b200.workloads import CONFIG_SHAPES, config_lengths  # noqa: E402

dev = torch.device("cuda:0")
lengths = config_lengths("c2")
hq, hkv, d, ps, _ = CONFIG_SHAPES["c2"]
pool, store, cfg = bench.build_cache(lengths, hq, hkv, d, ps, extra_tokens=400, device=dev)
B = len(lengths)
batch = DecodeBatch(store, list(range(B)), cfg)
q = torch.randn((B, hq, d)).bfloat16().pin_memory()
k = torch.randn((B, hkv, d)).bfloat16().pin_memory()
oh = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()
lib = _lib.load()
ph = {"call": [], "total": [], "after_call_sync": []}
for i in range(80):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batch.step(q, k, k, out=oh)
    t1 = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    t2 = time.perf_counter()
    if i >= 20:
        ph["call"].append((t1 - t0) * 1e6)
        ph["total"].append((t2 - t0) * 1e6)
        ph["after_call_sync"].append((t2 - t1) * 1e6)
print({kk: round(float(np.median(v)), 1) for kk, v in ph.items()})
# pieces
T = {"inputs": [], "stage_setup": [], "native": [], "finish": []}
n = B
for i in range(60):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batch._keep = []
    qq, qh, qb = batch._input(q, torch.bfloat16, (n, hq, d), "queries")
    kk, kh, kb = batch._input(k, store.torch_dtype, (n, hkv, d), "k_new")
    vv, vh, _ = batch._input(k, store.torch_dtype, (n, hkv, d), "v_new")
    o = batch._buffer("out", (n, hq, d), torch.float32)
    t1 = time.perf_counter()
    slot = batch._stage_setup()
    a = batch._args
    a.q, a.q_dtype = qq.data_ptr(), _lib.PKV_BF16
    a.k_cache, a.v_cache = store.keys.data_ptr(), store.values.data_ptr()
    a.kv_dtype, a.page_size = store.dtype_code, ps
    a.block_table, a.bt_stride = batch._stage.mirror_dev, batch._stage.mirror_cols
    a.out, a.out_dtype, a.mode = o.data_ptr(), _lib.PKV_F32, 0
    a.k_new, a.v_new = kk.data_ptr(), vv.data_ptr()
    io = batch._io
    io.q_host, io.k_host, io.v_host, io.q_bytes, io.kv_bytes = qh, kh, vh, qb, kb
    io.out_host, io.out_bytes = oh.data_ptr(), oh.numel() * 4
    t2 = time.perf_counter()
    st = lib.pkv_decode_step(batch._stage_p, batch._args_p, batch._io_p, _stream(dev))
    t3 = time.perf_counter()
    batch._stage_finish(slot)
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    if i >= 10:
        for key, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
            T[key].append(v * 1e6)
print({kk: round(float(np.median(v)), 1) for kk, v in T.items()})
# the host planner alone at this step's lengths
nk = np.asarray([pool.table(s).logical_len + 1 for s in range(B)], dtype=np.int32)
rows = np.arange(B, dtype=np.int32)
cap = lib.pkv_attention_plan_ints(B, hq)
plan = np.zeros(cap, dtype=np.int32)
got = C.c_int64()
t0 = time.perf_counter()
for _ in range(200):
    lib.pkv_attention_plan(nk.ctypes.data, rows.ctypes.data, B, ps, hq, hkv, 0, 0, plan.ctypes.data, cap,
                           C.byref(got))
print("plan us", round((time.perf_counter() - t0) / 200 * 1e6, 1))
# raw CUDA costs
s = torch.cuda.current_stream()
x = torch.empty(1 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    y[:4096].copy_(x[:4096], non_blocking=True)
print("torch h2d issue us", round((time.perf_counter() - t0) / 200 * 1e6, 1))
torch.cuda.synchronize()
