"""Per-line host timing of DecodeBatch.step(advance=False) (diagnostic)."""
import os, sys, time, ctypes as C
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2506_07311_b200 import _lib
from paper_2506_07311_b200.batch import DecodeBatch, PRECISION_MODES
from paper_2506_07311_b200.store import _stream, torch_dtype
from paper_2506_07311_b200.workloads import CONFIG_SHAPES, config_lengths
dev = torch.device("cuda:0")
lengths = config_lengths("c2")
hq, hkv, d, ps, _ = CONFIG_SHAPES["c2"]
pool, store, cfg = bench.build_cache(lengths, hq, hkv, d, ps, extra_tokens=200, device=dev)
B = len(lengths)
self = DecodeBatch(store, list(range(B)), cfg)
qd = torch.randn((B, hq, d), device=dev).bfloat16(); kd = torch.randn((B, hkv, d), device=dev).bfloat16()
T = {}
def tick(name, t):
    T.setdefault(name, []).append((time.perf_counter_ns() - t) / 1e3)
    return time.perf_counter_ns()
for it in range(50):
    torch.cuda.synchronize()
    t = time.perf_counter_ns()
    self.prepare(); t = tick("prepare", t)
    host, dev_m, done = self._ring[self._cur]; t = tick("ring", t)
    mirror = self.pool.device_table(self.device); t = tick("device_table", t)
    k = kd; v = kd
    ok = k.device != self.device or k.dtype != store.torch_dtype or not k.is_contiguous(); t = tick("kchecks", t)
    q, qcode = qd, self._qcodes[qd.dtype]; t = tick("q", t)
    out_t, out_code = torch_dtype(torch.float32); t = tick("torch_dtype", t)
    out = torch.empty((B, hq, d), dtype=out_t, device=self.device); t = tick("empty", t)
    md = dev_m.data_ptr(); hp = host.data_ptr(); t = tick("data_ptr", t)
    a = self._args
    a.q, a.q_dtype = q.data_ptr(), qcode
    a.q_seq, a.q_nkeys, a.seq_row = md, md + 4 * B, md + 8 * B
    a.k_cache, a.v_cache, a.kv_dtype = store.keys.data_ptr(), store.values.data_ptr(), store.dtype_code
    a.block_table, a.bt_stride = mirror.data_ptr(), mirror.shape[1]
    a.page_size = store.page_size
    a.out, a.out_dtype = out.data_ptr(), out_code
    a.workspace, a.workspace_bytes = self._ws.data_ptr(), self._ws.numel()
    a.mode = PRECISION_MODES["auto"]
    a.k_new, a.v_new = k.data_ptr(), v.data_ptr()
    a.plan, a.plan_host = md + 12 * B, hp + 12 * B
    a.meta_host = hp; a.meta_dev = md; a.meta_bytes = 4 * self._used.value; t = tick("args", t)
    sp = _stream(self.device); t = tick("stream", t)
    st = self._lib.pkv_paged_attention(self._args_p, sp); t = tick("launch", t)
    done.record(); t = tick("record", t)
print({k: round(float(np.median(v[10:])), 1) for k, v in T.items()})
