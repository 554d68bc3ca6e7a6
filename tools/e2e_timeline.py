"""Where one public-API decode step (DecodeBatch.step on C2, pinned host
q/k/v in, pinned host output) spends its wall time: host clock
(CLOCK_REALTIME ns) around the call next to the decode kernel's own
globaltimer stamps (first CTA start, last CTA end; pkv_debug_trace).  The
GPU's globaltimer follows the host's realtime clock; a calibration kernel
(empty torch op bracketed by host stamps) bounds the offset."""
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
from paper_2506_07311_b200.workloads import CONFIG_SHAPES, config_lengths  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
if os.environ.get("C3"):  # C3 point: "B:CTX"
    b3, ctx3 = (int(x) for x in os.environ["C3"].split(":"))
    lengths = [ctx3] * b3
    hq, hkv, d, ps, _ = CONFIG_SHAPES["c3"]
else:
    lengths = config_lengths("c2")
    hq, hkv, d, ps, _ = CONFIG_SHAPES["c2"]
pool, store, cfg = bench.build_cache(lengths, hq, hkv, d, ps, extra_tokens=200, device=dev)
B = len(lengths)
batch = DecodeBatch(store, list(range(B)), cfg)
rng = np.random.default_rng(7)
q = torch.from_numpy(rng.standard_normal((B, hq, d)).astype(np.float32)).bfloat16().pin_memory()
k = torch.from_numpy(rng.standard_normal((B, hkv, d)).astype(np.float32)).bfloat16().pin_memory()
v = torch.from_numpy(rng.standard_normal((B, hkv, d)).astype(np.float32)).bfloat16().pin_memory()
out = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()
flush = torch.ones(64 << 20, device=dev)
stream = torch.cuda.current_stream(dev)
lib = _lib.load()
for _ in range(8):
    batch.step(q, k, v, out=out)
torch.cuda.synchronize()
n = 256 * 8 * 32
rows, nat = [], []
st = (C.c_int64 * 12)()
for i in range(int(os.environ.get("STEPS", "12"))):
    flush.sum()
    torch.cuda.synchronize()
    lib.pkv_debug_trace(1, None, 0)
    m0 = time.monotonic_ns()
    t0 = time.time_ns()
    batch.step(q, k, v, out=out)
    t1 = time.time_ns()
    lib.pkv_debug_step_times(st, 12)
    entry = st[11] - m0  # python before the native call (steady clock == CLOCK_MONOTONIC)
    nat.append([entry / 1e3] + [st[j] / 1e3 for j in range(11)])
    stream.synchronize()
    t2 = time.time_ns()
    buf = (C.c_uint64 * n)()
    lib.pkv_debug_trace(-1, buf, n)
    lib.pkv_debug_trace(0, None, 0)
    t = np.array(buf, dtype=np.float64).reshape(256, 8, 32)
    starts = t[:, :, 0][t[:, :, 0] > 0]
    ends = t[:, :, 31][t[:, :, 31] > 0]
    ks, ke = starts.min(), ends.max()
    rows.append(((ks - t0) / 1e3, (ke - ks) / 1e3, (t2 - ke) / 1e3, (t1 - t0) / 1e3, (t2 - t0) / 1e3))
r = np.array(rows)
names = ("call start -> first CTA", "kernel span", "last CTA end -> sync returns", "host time in step()",
         "wall per step")
for j, nm in enumerate(names):
    print("%-32s median %7.1f us  min %7.1f  max %7.1f" % (nm, np.median(r[:, j]), r[:, j].min(), r[:, j].max()))

nat = np.array(nat)
print("python before native call: median %.1f us" % np.median(nat[:, 0]))
labels = {1: "input H2D issued", 2: "slot event", 3: "allocator+plan", 7: "stage done (upload, aux)",
          8: "decode launched", 9: "output D2H issued", 10: "next plan speculated"}
for j, lab in labels.items():
    print("  native stamp %2d %-26s median %6.1f us after entry" % (j, lab, np.median(nat[:, j + 1])))

# calibration: the same measurement on a tiny decode (1 sequence x 64 keys):
# its "last CTA end -> sync returns" is the wake-up floor plus the clock
# offset, which cancels in the difference with the C2 step above
pool2, store2, cfg2 = bench.build_cache([64], hq, hkv, d, ps, extra_tokens=200, device=dev)
b2 = DecodeBatch(store2, [0], cfg2)
q2 = torch.zeros((1, hq, d), dtype=torch.bfloat16).pin_memory()
k2 = torch.zeros((1, hkv, d), dtype=torch.bfloat16).pin_memory()
o2 = torch.empty((1, hq, d), dtype=torch.float32).pin_memory()
for _ in range(5):
    b2.step(q2, k2, k2, out=o2)
torch.cuda.synchronize()
cal = []
for i in range(12):
    torch.cuda.synchronize()
    lib.pkv_debug_trace(1, None, 0)
    t0 = time.time_ns()
    b2.step(q2, k2, k2, out=o2)
    stream.synchronize()
    t2 = time.time_ns()
    buf = (C.c_uint64 * n)()
    lib.pkv_debug_trace(-1, buf, n)
    lib.pkv_debug_trace(0, None, 0)
    t = np.array(buf, dtype=np.float64).reshape(256, 8, 32)
    ks = t[:, :, 0][t[:, :, 0] > 0].min()
    ke = t[:, :, 31][t[:, :, 31] > 0].max()
    cal.append(((ks - t0) / 1e3, (ke - ks) / 1e3, (t2 - ke) / 1e3, (t2 - t0) / 1e3))
cal = np.array(cal)
pre_d = np.median(r[:, 0]) - np.median(cal[:, 0])
post_d = np.median(r[:, 2]) - np.median(cal[:, 2])
print("tiny decode: wall %.1f us, span %.1f us" % (np.median(cal[:, 3]), np.median(cal[:, 1])))
print("C2 minus tiny: call->first CTA %+.1f us, last CTA->sync %+.1f us" % (pre_d, post_d))
