import time, sys, os, ctypes as C
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2506_07311_b200 import KvStore, PagePool, _lib
from paper_2506_07311_b200.store import _stream, to_device
dev = torch.device("cuda:0")
n, hkv, d, ps = 8192, 8, 128, 16
pool = PagePool(n // ps + 8, page_size=ps)
store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=dev)
pool.reserve(0, n)
k = torch.randn((n, hkv, d), device=dev).bfloat16()
pos = np.arange(n)
for _ in range(5): store.assign(0, pos, k, k)
torch.cuda.synchronize()
def t(fn, reps=50):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); out.append((time.perf_counter() - t0) * 1e6)
    return round(float(np.median(out)), 1)
table = pool.table(0)
info, copies, cnt = store._assign_scratch(n)
lib = _lib.load()
mirror = pool.device_table(dev)
def prep():
    lib.pkv_pool_assign_prepare(pool._h, table._handle, pos.ctypes.data, n, info.ctypes.data, copies.ctypes.data, copies.size, C.addressof(cnt))
def launch():
    lib.pkv_kv_append_range(k.data_ptr(), k.data_ptr(), n, 0, 0, mirror.data_ptr(), mirror.shape[1], ps, store._k_ptr, store._v_ptr, store.row_bytes, _stream(dev))
ev = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); launch(); b.record(); torch.cuda.synchronize(); ev.append(a.elapsed_time(b) * 1e3)
print({"table": t(lambda: pool.table(0)), "asarray": t(lambda: np.ascontiguousarray(np.asarray(pos, dtype=np.int64))),
       "prepare": t(prep), "to_device": t(lambda: to_device(k, dev, torch.bfloat16)),
       "device_table": t(lambda: pool.device_table(dev)), "stream": t(lambda: _stream(dev)),
       "launch_host": t(launch), "kernel_us_p50": round(float(np.median(ev)), 1),
       "logical_len_set": t(lambda: setattr(table, "logical_len", n)),
       "assign_total": t(lambda: store.assign(0, pos, k, k))})
