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

    def __init__(self, stores, seq_ids, config: AttentionConfig, capacity: int | None = None):
        import torch

        self.stores = list(stores) if isinstance(stores, (list, tuple)) else [stores]
        self.pool = self.stores[0].pool
        self.device = self.stores[0].device
        if any(s.pool is not self.pool for s in self.stores):
            raise ValueError("all stores of a DecodeBatch must share one pool")
        self.config = config
        self._lib = _lib.load()
        self._qcodes = {torch.float32: _lib.PKV_F32, torch.float16: _lib.PKV_F16,
                        torch.bfloat16: _lib.PKV_BF16}
        self._used = C.c_int64()
        self._used_p = C.byref(self._used)
        self._n_pages = C.c_int64()
        self._n_pages_p = C.byref(self._n_pages)
        self._cap = 0
        self.last_launches = 0
        # one persistent argument block; step() updates the per-call fields
        self._args = _lib.AttentionArgs(
            seq_start=None, hq=config.head_count, hkv=config.kv_head_count, head_dim=config.head_dim,
            scale=float(config.scale), num_sms=0, target_waves=0, prof_start=None, prof_stop=None)
        self._args_p = C.byref(self._args)
        self.set_sequences(seq_ids, capacity)

    def set_sequences(self, seq_ids, capacity: int | None = None) -> None:
        """Change the batch membership (continuous batching): later steps
        advance exactly these sequences.  Staging buffers are reused while
        the batch fits the current capacity and regrown (x2) otherwise."""
        import torch

        self.seq_ids = list(seq_ids)
        self.n = len(self.seq_ids)
        self.handles = np.asarray([self.pool.table(s)._handle for s in self.seq_ids], dtype=np.int64)
        self._handles_p = self.handles.ctypes.data_as(C.POINTER(C.c_int64))
        need = max(self.n, int(capacity or 0), 1)
        if need > self._cap:
            cap = max(need, 2 * self._cap)
            cfg = self.config
            self._copies = np.empty(2 * cap, dtype=np.int64)
            self._pages = np.empty(2 * cap + 1, dtype=np.uint32)
            self._pages_p = self._pages.ctypes.data_as(C.POINTER(C.c_uint32))
            self._copies_p = self._copies.ctypes.data_as(C.POINTER(C.c_int64))
            # packed per-step metadata [q_seq | nkeys | rows | plan]: a ring of
            # pinned staging buffers, each reused only after its upload landed
            width = 3 * cap + int(self._lib.pkv_attention_plan_ints(cap, cfg.head_count))
            self._ring = []
            for _ in range(4):
                host = torch.empty(width, dtype=torch.int32).pin_memory()
                dev = torch.empty(width, dtype=torch.int32, device=self.device)
                self._ring.append((host, dev, torch.cuda.Event()))
            ws_bytes = self._lib.pkv_attention_workspace_bytes(cap, cfg.head_count, cfg.head_dim)
            self._ws = _Workspace.get(self.device, ws_bytes)
            self._cap = cap
        self._slot = 0
        self._cur = None
        self._uploaded = False
        self._args.n_queries = self.n

    def prepare(self) -> int:
        """Host work of one token step: one native call does the allocator
        bookkeeping (grow, copy-on-write, logical_len) and writes the packed
        metadata [q_seq | nkeys | rows | plan] into a pinned staging slot.
        Returns the number of page clear/copy launches it caused."""
        if self.n == 0:
            raise ValueError("the decode batch is empty")
        slot = self._slot
        self._slot = (slot + 1) % len(self._ring)
        host, dev, done = self._ring[slot]
        done.synchronize()  # the previous upload from this slot has landed
        cfg = self.config
        st = self._lib.pkv_decode_step_prepare(
            self.pool._h, self._handles_p, self.n, self.pool.page_size, cfg.head_count, cfg.kv_head_count,
            host.data_ptr(), host.numel(), self._used_p, self._pages_p, self._pages.size, self._n_pages_p,
            self._copies_p)
        if st:
            _lib.check(st, "pkv_decode_step_prepare")
        self._cur = slot
        self._uploaded = False
        launches = 0
        n_pages = self._n_pages.value
        if n_pages:
            self.pool._clear_pages(self._pages[:n_pages].tolist())
            launches += len(self.pool._stores)
        pairs = self._copies[: 2 * self.n].reshape(-1, 2)
        cow = pairs[:, 1] >= 0
        if cow.any():  # copy-on-write pages: one batched K0b launch per store
            sel = pairs[cow]
            self.pool._copy_pages(np.column_stack([sel, np.full(len(sel), self.pool.page_size)]))
            launches += len(self.pool._stores)
        return launches

    def step(self, queries, k_new, v_new, *, out_dtype=None, layer: int = 0, advance: bool = True,
             precision: str = "auto"):
        """Append one token per sequence into `stores[layer]` and attend.

        queries [B, Hq, D]; k_new / v_new [B, Hkv, D] (numpy or torch, any
        device)."""
        import torch

        launches = self.prepare() if advance else 0
        if self._cur is None:
            raise ValueError("call prepare() before step(advance=False)")
        store: KvStore = self.stores[layer]
        cfg = self.config
        n = self.n
        host, dev, done = self._ring[self._cur]
        mirror = self.pool.device_table(self.device)  # applies any pending table edits
        k = k_new if isinstance(k_new, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(k_new))
        v = v_new if isinstance(v_new, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v_new))
        if k.device != self.device or k.dtype != store.torch_dtype or not k.is_contiguous():
            k = k.to(device=self.device, dtype=store.torch_dtype, non_blocking=True).contiguous()
        if v.device != self.device or v.dtype != store.torch_dtype or not v.is_contiguous():
            v = v.to(device=self.device, dtype=store.torch_dtype, non_blocking=True).contiguous()
        if isinstance(queries, torch.Tensor) and queries.device == self.device and queries.is_contiguous() \
                and queries.dtype in self._qcodes:
            q, qcode = queries, self._qcodes[queries.dtype]
        else:
            q, qcode = _q_tensor(queries, self.device)
        out_t, out_code = torch_dtype(out_dtype or torch.float32)
        out = torch.empty((n, cfg.head_count, cfg.head_dim), dtype=out_t, device=self.device)
        md = dev.data_ptr()
        hp = host.data_ptr()
        a = self._args
        a.q, a.q_dtype = q.data_ptr(), qcode
        a.q_seq, a.q_nkeys, a.seq_row = md, md + 4 * n, md + 8 * n
        a.k_cache, a.v_cache, a.kv_dtype = store.keys.data_ptr(), store.values.data_ptr(), store.dtype_code
        a.block_table, a.bt_stride = mirror.data_ptr(), mirror.shape[1]
        a.page_size = store.page_size
        a.out, a.out_dtype = out.data_ptr(), out_code
        a.workspace, a.workspace_bytes = self._ws.data_ptr(), self._ws.numel()
        a.mode = PRECISION_MODES[precision]
        a.k_new, a.v_new = k.data_ptr(), v.data_ptr()
        a.plan, a.plan_host = md + 12 * n, hp + 12 * n
        # the first layer of a token uploads the packed metadata on the stream
        a.meta_host = None if self._uploaded else hp
        a.meta_dev = md
        a.meta_bytes = 4 * self._used.value
        # K1 append is fused into the decode launch (the last split of every
        # sequence reads the new token from k/v and writes it into its page)
        st = self._lib.pkv_paged_attention(self._args_p, _stream(self.device))
        if st:
            _lib.check(st, "pkv_paged_attention")
        if not self._uploaded:
            done.record()
            self._uploaded = True
        tensor = (store.dtype_code == _lib.PKV_BF16 and precision != "exact") or precision == "tensor"
        # tensor-core path: one launch (append fused, split merge in-kernel)
        self.last_launches = launches + (1 if tensor else 4)
        return out
