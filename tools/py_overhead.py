import sys, time, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2506_07311_b200.batch import DecodeBatch
from paper_2506_07311_b200 import _lib
from paper_2506_07311_b200.store import _stream
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
_, lengths, hq, hkv, d, ps = bench.workload("c2", 0, 1)
pool, store, cfg = bench.build_cache(lengths, hq, hkv, d, ps, extra_tokens=2000, device=dev)
B = len(lengths)
batch = DecodeBatch(store, list(range(B)), cfg)
q, k, v = DecodeBatch.packed_host_inputs(B, hq, hkv, d, torch.bfloat16)
oh = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()
def t(name, fn, n=2000):
    fn()
    t0 = time.perf_counter_ns()
    for _ in range(n): fn()
    print(f"{name}: {(time.perf_counter_ns()-t0)/n/1e3:.2f} us")
t("current_device", torch.cuda.current_device)
t("current_stream", lambda: torch.cuda.current_stream(dev))
t("_stream", lambda: _stream(dev))
a = batch._args
def sets():
    a.q = 123; a.k_new = 456; a.v_new = 789; a.out = 1000; a.mode = 0
t("5 ctypes sets", sets)
t("_input", lambda: batch._input(q, torch.bfloat16, (B, hq, d), "queries"))
t("_native_pages", batch._native_pages)
t("data_ptr", q.data_ptr)
t("is_pinned", q.is_pinned)
t("stage_setup", batch._stage_setup)
t("isinstance", lambda: isinstance(q, torch.Tensor))
t("shape tuple", lambda: tuple(q.shape) == (B, hq, d))
st = torch.cuda.current_stream(dev)
def full():
    batch.step(q, k, v, out=oh)
for i in range(20): full(); st.synchronize()
ts = []
for i in range(200):
    t0 = time.perf_counter_ns(); full(); ts.append(time.perf_counter_ns()-t0); st.synchronize()
print("step host us median", np.median(ts)/1e3)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for i in range(200): full(); st.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(12)
