"""C2 e2e step decomposed: where do the host/PCIe microseconds go?

Variants of DecodeBatch.step on the bench's C2 cache (all synchronous per
step, L2 flushed, median of 40):
  full      pinned host q/k/v in, pinned host out (the bench's e2e)
  dev_in    device-resident q/k/v, pinned host out
  dev_out   pinned host q/k/v in, device out
  dev_all   device in / device out (the API path without PCIe)
  host_only time until step() returns (no sync), full variant
Run with PKV_ZERO_COPY_IN=1 to read host q/k/v through mapped pointers."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_07311_b200.batch import DecodeBatch  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
_, lengths, hq, hkv, d, ps = bench.workload(cfgname, 0, 1)
pool, store, cfg = bench.build_cache(lengths, hq, hkv, d, ps, extra_tokens=2000, device=dev)
B = len(lengths)
batch = DecodeBatch(store, list(range(B)), cfg)
flush = bench.L2Flush(dev)
qh = torch.randn((B, hq, d)).bfloat16().pin_memory()
kh = torch.randn((B, hkv, d)).bfloat16().pin_memory()
vh = torch.randn((B, hkv, d)).bfloat16().pin_memory()
qp, kp, vp = DecodeBatch.packed_host_inputs(B, hq, hkv, d, torch.bfloat16)
qp.copy_(qh), kp.copy_(kh), vp.copy_(vh)
oh = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()
qd, kd, vd = qh.to(dev), kh.to(dev), vh.to(dev)
od = torch.empty((B, hq, d), dtype=torch.float32, device=dev)
st = torch.cuda.current_stream(dev)
res = {}
for name, (q, k, v, o) in {"full": (qh, kh, vh, oh), "packed": (qp, kp, vp, oh), "dev_in": (qd, kd, vd, oh), "dev_out": (qh, kh, vh, od),
                           "dev_all": (qd, kd, vd, od)}.items():
    ts, th = [], []
    for i in range(50):
        flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        batch.step(q, k, v, out=o)
        t1 = time.perf_counter()
        st.synchronize()
        t2 = time.perf_counter()
        if i >= 10:
            ts.append((t2 - t0) * 1e6)
            th.append((t1 - t0) * 1e6)
    res[name] = (round(float(np.median(ts)), 1), round(float(np.median(th)), 1))
kv = sum(2 * (n + 100) * hkv * d * 2 for n in lengths)
print(cfgname, "zero_copy_in" if os.environ.get("PKV_ZERO_COPY_IN") == "1" else "h2d",
      {k: {"step_us": v[0], "host_return_us": v[1], "TB/s": round(kv / v[0] / 1e6, 2)} for k, v in res.items()})

# native phase stamps of the full variant (median over steps, microseconds)
import ctypes as C  # noqa: E402

from paper_2506_07311_b200 import _lib  # noqa: E402

lib = _lib.load()
buf = (C.c_int64 * 12)()
rows = []
for i in range(40):
    flush()
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns()
    batch.step(qp, kp, vp, out=oh)
    t1 = time.perf_counter_ns()
    st.synchronize()
    t2 = time.perf_counter_ns()
    lib.pkv_debug_step_times(buf, 12)
    entry = (buf[11] - t0) / 1e3
    rows.append([entry] + [entry + x / 1e3 for x in buf[0:11]] + [(t1 - t0) / 1e3, (t2 - t0) / 1e3])
med = np.median(np.asarray(rows[10:]), axis=0)
names = ["py_to_native", "device_guard", "h2d_issued", "slot_free", "alloc_plan", "side", "meta_upload", "aux", "pre_launch",
         "launched", "out_copy", "speculated", "py_return", "synced"]
print("packed, us since step() entry:", {n: round(float(v), 1) for n, v in zip(names, med)})

# device-side split per variant: [step issue -> kernel start] (H2D +
# metadata + aux), kernel, [kernel end -> step end]
for name, (q, k, v, o) in {"packed": (qp, kp, vp, oh), "dev_out": (qp, kp, vp, od),
                           "dev_all": (qd, kd, vd, od)}.items():
    evs = []
    for i in range(40):
        e0, ks, ke, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        for e in (ks, ke):
            e.record()
        flush()
        torch.cuda.synchronize()
        e0.record()
        batch._args.prof_start, batch._args.prof_stop = ks.cuda_event, ke.cuda_event
        batch.step(q, k, v, out=o)
        e1.record()
        st.synchronize()
        evs.append((e0.elapsed_time(ks) * 1e3, ks.elapsed_time(ke) * 1e3, ke.elapsed_time(e1) * 1e3,
                    e0.elapsed_time(e1) * 1e3))
    batch._args.prof_start = batch._args.prof_stop = None
    med = np.median(np.asarray(evs[10:]), axis=0)
    print(name, {"issue_to_kernel_us": round(float(med[0]), 1), "kernel_us": round(float(med[1]), 1),
                 "kernel_to_end_us": round(float(med[2]), 1), "device_total_us": round(float(med[3]), 1)})
