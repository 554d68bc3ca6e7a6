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
        self._cap = 0
        self.last_launches = 0
        # one persistent argument block; step() updates the per-call fields
        self._args = _lib.AttentionArgs(
            seq_start=None, hq=config.head_count, hkv=config.kv_head_count, head_dim=config.head_dim,
            scale=float(config.scale), num_sms=0, target_waves=0, prof_start=None, prof_stop=None)
        self._args_p = C.byref(self._args)
        self._stage = _lib.StepStageArgs()
        self._stage_p = C.byref(self._stage)
        self._stage_stores = None
        self._store_ptrs = {}
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
            # packed per-step metadata [q_seq | nkeys | rows | plan]: a ring of
            # pinned staging buffers, each reused only after its upload landed
            width = int(self._lib.pkv_decode_step_stage_ints(cap, cfg.head_count))
            self._ring = []
            for _ in range(4):
                host = torch.empty(width, dtype=torch.int32).pin_memory()
                dev = torch.empty(width, dtype=torch.int32, device=self.device)
                ev = torch.cuda.Event()
                ev.record()  # materialise the cudaEvent_t handle
                self._ring.append((host, dev, ev))
            ws_bytes = self._lib.pkv_attention_workspace_bytes(cap, cfg.head_count, cfg.head_dim)
            self._ws = _Workspace.get(self.device, ws_bytes)
            self._args.workspace, self._args.workspace_bytes = self._ws.data_ptr(), self._ws.numel()
            self._cap = cap
        self._slot = 0
        self._cur = None
        self._args.n_queries = self.n

    def prepare(self, _sp=None) -> int:
        """Host work of one token step in one native call
        (pkv_decode_step_stage): allocator bookkeeping (grow, copy-on-write,
        logical_len), the packed metadata + work plan, their upload, the page
        clears / copies in every attached store and the block-table mirror
        update.  Returns the number of auxiliary kernels it launched."""
        if self.n == 0:
            raise ValueError("the decode batch is empty")
        slot = self._slot
        self._slot = (slot + 1) % len(self._ring)
        host, dev, done = self._ring[slot]
        stores = self.pool._stores
        row_bytes = {s.row_bytes for s in stores}
        native_pages = len(row_bytes) == 1
        if native_pages and self._stage_stores != [id(s) for s in stores]:
            self._kc = (C.c_void_p * len(stores))(*[s.keys.data_ptr() for s in stores])
            self._vc = (C.c_void_p * len(stores))(*[s.values.data_ptr() for s in stores])
            self._stage_stores = [id(s) for s in stores]
        mirror = self.pool._mirror
        if mirror is None or mirror.device != self.device:
            mirror = self.pool.device_table(self.device)
        a = self._stage
        a.pool, a.seqs, a.n = self.pool._h, self.handles.ctypes.data, self.n
        a.page_size, a.hq, a.hkv = self.pool.page_size, self.config.head_count, self.config.kv_head_count
        a.meta_host, a.meta_dev, a.meta_cap = host.data_ptr(), dev.data_ptr(), host.numel()
        a.slot_event = done.cuda_event
        a.n_stores = len(stores) if native_pages else 0
        a.k_caches = C.cast(self._kc, C.c_void_p) if native_pages else None
        a.v_caches = C.cast(self._vc, C.c_void_p) if native_pages else None
        a.row_bytes = next(iter(row_bytes)) if native_pages else 0
        a.mirror_dev, a.mirror_rows, a.mirror_cols = mirror.data_ptr(), mirror.shape[0], mirror.shape[1]
        st = self._lib.pkv_decode_step_stage(self._stage_p, _sp if _sp is not None else _stream(self.device))
        if st:
            _lib.check(st, "pkv_decode_step_stage")
        launches = a.launches
        if not native_pages:  # stores of different row sizes: page work through the stores
            meta = host.numpy()
            if a.n_granted:
                self.pool._clear_pages(meta[a.granted_off:a.granted_off + a.n_granted].tolist())
                launches += len(stores)
            if a.n_copies:
                self.pool._copy_pages(meta[a.copies_off:a.copies_off + 3 * a.n_copies].reshape(-1, 3))
                launches += len(stores)
        if a.needs_resync:
            self.pool.device_table(self.device)  # shape change: full re-export
        self._cur = slot
        self._used.value = a.meta_used
        return launches

    def step(self, queries, k_new, v_new, *, out_dtype=None, layer: int = 0, advance: bool = True,
             precision: str = "auto"):
        """Append one token per sequence into `stores[layer]` and attend.

        queries [B, Hq, D]; k_new / v_new [B, Hkv, D] (numpy or torch, any
        device)."""
        import torch

        sp = _stream(self.device)
        launches = self.prepare(sp) if advance else 0
        if self._cur is None:
            raise ValueError("call prepare() before step(advance=False)")
        store: KvStore = self.stores[layer]
        cfg = self.config
        n = self.n
        host, dev, done = self._ring[self._cur]
        mirror = self.pool.device_table(self.device)  # applies any pending table edits
        kv_t = store.torch_dtype
        k = k_new if isinstance(k_new, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(k_new))
        v = v_new if isinstance(v_new, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v_new))
        if k.device != self.device or k.dtype != kv_t or not k.is_contiguous():
            k = k.to(device=self.device, dtype=kv_t, non_blocking=True).contiguous()
        if v.device != self.device or v.dtype != kv_t or not v.is_contiguous():
            v = v.to(device=self.device, dtype=kv_t, non_blocking=True).contiguous()
        if isinstance(queries, torch.Tensor) and queries.device == self.device and queries.is_contiguous() \
                and queries.dtype in self._qcodes:
            q, qcode = queries, self._qcodes[queries.dtype]
        else:
            q, qcode = _q_tensor(queries, self.device)
        out_t, out_code = (torch.float32, _lib.PKV_F32) if out_dtype is None else torch_dtype(out_dtype)
        out = torch.empty((n, cfg.head_count, cfg.head_dim), dtype=out_t, device=self.device)
        md = dev.data_ptr()
        hp = host.data_ptr()
        ptrs = self._store_ptrs.get(id(store))
        if ptrs is None:
            ptrs = (store.keys.data_ptr(), store.values.data_ptr(), store.dtype_code, store.page_size)
            self._store_ptrs[id(store)] = ptrs
        a = self._args
        a.q, a.q_dtype = q.data_ptr(), qcode
        a.q_seq, a.q_nkeys, a.seq_row = md, md + 4 * n, md + 8 * n
        a.k_cache, a.v_cache, a.kv_dtype, a.page_size = ptrs
        a.block_table, a.bt_stride = mirror.data_ptr(), mirror.shape[1]
        a.out, a.out_dtype = out.data_ptr(), out_code
        a.mode = PRECISION_MODES[precision]
        a.k_new, a.v_new = k.data_ptr(), v.data_ptr()
        a.plan, a.plan_host = md + 12 * n, hp + 12 * n
        a.meta_host = None  # uploaded by prepare() (pkv_decode_step_stage)
        a.meta_dev = md
        a.meta_bytes = 0
        # K1 append is fused into the decode launch (the last split of every
        # sequence reads the new token from k/v and writes it into its page)
        st = self._lib.pkv_paged_attention(self._args_p, sp)
        if st:
            _lib.check(st, "pkv_paged_attention")
        tensor = (store.dtype_code == _lib.PKV_BF16 and precision != "exact") or precision == "tensor"
        # tensor-core path: one launch (append fused, split merge in-kernel)
        self.last_launches = launches + (1 if tensor else 4)
        return out
