"""Batched decode step — B sequences advance one token through one
allocator call, one metadata upload and one decode launch (+ the split
combine when a sequence is split).

This is the serving-loop form of the reference's per-session
`DecodeSession.step` (decoder.py:263-284): grow -> assign at `logical_len`
-> attend over all `logical_len + 1` keys (the new token included,
attention.py:86-96).  Semantics per sequence are exactly the reference's; the
batch only amortises host work (one native `pkv_pool_prepare_append` for all
allocator bookkeeping, the host work plan, one packed metadata upload) and
launches: the K1 append is fused into the K2 launch.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .attention import PRECISION_MODES, AttentionConfig, _Workspace, _q_tensor
from .store import KvStore, _stream, torch_dtype


class DecodeBatch:
    """Decode B sequences of one pool together.

    `stores` is one KvStore (one layer) or a list of stores on the same pool
    (one per layer): call `prepare()` once per token, then
    `step(..., layer=i, advance=False)` for every layer (or just `step(...)`
    for a single layer).
    """

    def __init__(self, stores, seq_ids, config: AttentionConfig):
        import torch

        self.stores = list(stores) if isinstance(stores, (list, tuple)) else [stores]
        self.pool = self.stores[0].pool
        self.device = self.stores[0].device
        if any(s.pool is not self.pool for s in self.stores):
            raise ValueError("all stores of a DecodeBatch must share one pool")
        self.config = config
        self.seq_ids = list(seq_ids)
        self.handles = np.asarray([self.pool.table(s)._handle for s in self.seq_ids], dtype=np.int64)
        self.n = len(self.seq_ids)
        self._pos = np.empty(self.n, dtype=np.int32)
        self._rows = np.empty(self.n, dtype=np.int32)
        self._copies = np.empty(2 * self.n, dtype=np.int64)
        self._pages = np.empty(2 * self.n + 1, dtype=np.uint32)
        self._plan_len = int(_lib.load().pkv_attention_plan_ints(self.n, config.head_count))
        # packed per-step metadata [q_seq | nkeys | rows | plan]: a ring of
        # pinned staging buffers, each reused only after its upload completed
        width = 3 * self.n + self._plan_len
        self._ring = []
        for _ in range(4):
            host = torch.empty(width, dtype=torch.int32).pin_memory()
            host[: self.n] = torch.arange(self.n, dtype=torch.int32)
            dev = torch.empty(width, dtype=torch.int32, device=self.device)
            self._ring.append((host, dev, torch.cuda.Event()))
        self._slot = 0
        self.last_launches = 0

    def prepare(self) -> int:
        """Allocator work of one token step (host, one native call); returns
        the number of page clear/copy launches it caused."""
        n_pages = C.c_int64()
        i64p, i32p, u32p = C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_uint32)
        _lib.call("pkv_pool_prepare_append", self.pool._h, self.handles.ctypes.data_as(i64p), self.n,
                  self._pos.ctypes.data_as(i32p), self._rows.ctypes.data_as(i32p),
                  self._pages.ctypes.data_as(u32p), self._pages.size, C.byref(n_pages),
                  self._copies.ctypes.data_as(i64p))
        launches = 0
        if n_pages.value:
            self.pool._clear_pages(self._pages[: n_pages.value].tolist())
            launches += len(self.pool._stores)
        for old, new in self._copies.reshape(-1, 2):
            if new >= 0:
                self.pool._copy_rows(int(old), int(new), self.pool.page_size)
                launches += len(self.pool._stores)
        return launches

    def step(self, queries, k_new, v_new, *, out_dtype=None, layer: int = 0, advance: bool = True,
             precision: str = "auto"):
        """Append one token per sequence into `stores[layer]` and attend.

        queries [B, Hq, D]; k_new / v_new [B, Hkv, D] (numpy or torch, any
        device)."""
        import torch

        launches = self.prepare() if advance else 0
        store: KvStore = self.stores[layer]
        cfg = self.config
        n = self.n
        host, dev, done = self._ring[self._slot]
        self._slot = (self._slot + 1) % len(self._ring)
        done.synchronize()  # the previous upload from this buffer has landed
        mh = host.numpy()
        nkeys = self._pos + 1  # keys attended: the whole context
        mh[n:2 * n] = nkeys
        mh[2 * n:3 * n] = self._rows
        plan = _lib.attention_plan(nkeys, self._rows, store.page_size, cfg.head_count, cfg.kv_head_count)
        used = 3 * n + plan.size
        mh[3 * n:used] = plan
        dev[:used].copy_(host[:used], non_blocking=True)
        done.record()
        mirror = self.pool.device_table(self.device)
        k = k_new if isinstance(k_new, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(k_new))
        v = v_new if isinstance(v_new, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v_new))
        k = k.to(device=self.device, dtype=store.torch_dtype, non_blocking=True).contiguous()
        v = v.to(device=self.device, dtype=store.torch_dtype, non_blocking=True).contiguous()
        md = dev.data_ptr()
        q, qcode = _q_tensor(queries, self.device)
        out_t, out_code = torch_dtype(out_dtype or torch.float32)
        out = torch.empty((n, cfg.head_count, cfg.head_dim), dtype=out_t, device=self.device)
        ws_bytes = _lib.load().pkv_attention_workspace_bytes(n, cfg.head_count, cfg.head_dim)
        ws = _Workspace.get(self.device, ws_bytes)
        args = _lib.AttentionArgs(
            q=q.data_ptr(), q_dtype=qcode, n_queries=n, q_seq=md, q_nkeys=md + 4 * n,
            k_cache=store.keys.data_ptr(), v_cache=store.values.data_ptr(), kv_dtype=store.dtype_code,
            block_table=mirror.data_ptr(), bt_stride=mirror.shape[1], seq_row=md + 8 * n,
            seq_start=None, page_size=store.page_size, hq=cfg.head_count, hkv=cfg.kv_head_count,
            head_dim=cfg.head_dim, scale=float(cfg.scale), out=out.data_ptr(), out_dtype=out_code,
            workspace=ws.data_ptr(), workspace_bytes=ws.numel(), num_sms=0, target_waves=0,
            mode=PRECISION_MODES[precision], k_new=k.data_ptr(), v_new=v.data_ptr(),
            plan=md + 12 * n, plan_host=host.data_ptr() + 12 * n)
        # K1 append is fused into the decode launch (the last split of every
        # sequence reads the new token from k/v and writes it into its page)
        _lib.check(_lib.load().pkv_paged_attention(C.byref(args), _stream(self.device)),
                   "pkv_paged_attention")
        tensor = (store.dtype_code == _lib.PKV_BF16 and precision != "exact") or precision == "tensor"
        split = int(mh[3 * n + 6]) > 0  # plan header: queries with > 1 split
        self.last_launches = launches + ((1 + split) if tensor else 4)
        return out
