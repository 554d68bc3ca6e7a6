"""Batched decode step — B sequences advance one token in ONE native call
(pkv_decode_step): host→device copies of CPU inputs, the allocator step,
the packed metadata + work plan upload, one aux kernel for page clears /
copies / block-table edits (only when pages are granted), and the decode
launch with the K1 append fused in; a pinned host output is written by the
kernel itself.  The next step's plan is computed while the GPU runs.

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
from .store import KvStore, _self_device, _stream, on_device, torch_dtype
from .errors import ShapeMismatch

import os as _os

# A pinned host `out` is written by the kernel itself through the mapped
# (UVA) host pointer instead of a trailing D2H copy: the stores stream over
# PCIe while the step runs (measured on C2: 196 -> 186 us per e2e step).
# PKV_ZERO_COPY_OUT=0 restores the copy.
_ZERO_COPY_OUT = _os.environ.get("PKV_ZERO_COPY_OUT", "1") != "0"
# Pinned host q / k_new / v_new read by the kernel through their mapped
# pointers (no H2D copy ahead of the launch).  Experiment switch.
_ZERO_COPY_IN = _os.environ.get("PKV_ZERO_COPY_IN", "0") == "1"
# Pinned host k_new / v_new only (the default): read by the kernel through
# their mapped pointers (the fused append and the new token's key row, 256-B
# coalesced reads spread over the launch), while the queries still go by DMA
# — the decode launch waits for the third of the inputs it needs first
# instead of all of them (C2 e2e 174-181 -> 160-161 us per step on a 20 GB/s
# PCIe box).  PKV_ZERO_COPY_KV=0 copies all three.
_ZERO_COPY_KV = _os.environ.get("PKV_ZERO_COPY_KV", "1") != "0"
# CUDA-graph mode of the repeated step (pkv_decode_step_graph): its kernels
# replayed as one cached graph.  Off by default (PKV_STEP_GRAPH=1 or
# DecodeBatch.use_graph turns it on): measured on C2 it saves ~4 us of host
# launch time but the graph executes ~10 us later on the GPU (host inputs:
# 165-172 vs 164 us per step; device inputs: 146-154 vs 137 us,
# tools/e2e_graph_ab.py), so the launch-by-launch step is faster.
_STEP_GRAPH = _os.environ.get("PKV_STEP_GRAPH", "0") == "1"


class _FastStep:
    """A repeatable step() call: the caller's buffers (held here, so their ids
    stay theirs) and private copies of the argument blocks the first call
    filled.  Valid while the same objects keep the same storage and the
    batch's membership, attached stores and staging buffers are unchanged."""

    __slots__ = ("tensors", "ptrs", "args", "args_p", "io", "io_p", "result", "out_host", "out_dev", "tensor",
                 "mirror", "fixed", "nstores", "bufs", "graph_ok")

    def __init__(self, batch, tensors, result, out_host, out_dev, tensor):
        self.tensors = tensors
        self.ptrs = tuple(t.data_ptr() for t in tensors)
        self.args = _lib.AttentionArgs.from_buffer_copy(batch._args)
        self.args_p = C.byref(self.args)
        self.io = _lib.DecodeIO.from_buffer_copy(batch._io)
        self.io_p = C.byref(self.io)
        self.result, self.out_host, self.out_dev, self.tensor = result, out_host, out_dev, tensor
        self.mirror = batch._stage_mirror
        self.fixed = batch._stage_fixed
        self.nstores = len(batch.pool._stores)
        self.bufs = batch._bufs
        # graph memcpy nodes need pinned (or device) sources and no host out copy
        self.graph_ok = out_host is None and all(
            t.is_cuda or t.is_pinned() for t in tensors[:3])

    def valid(self, batch, q, k, v, out) -> bool:
        t = self.tensors
        return (q is t[0] and k is t[1] and v is t[2] and out is t[3] and self.bufs is batch._bufs
                and self.fixed == batch._stage_fixed and self.nstores == len(batch.pool._stores)
                and (q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr()) == self.ptrs)


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
        self._uniform = False
        self._stage_fixed = None
        self._stage_mirror = None
        self._io = _lib.DecodeIO()
        self._io_p = C.byref(self._io)
        self._bufs = {}
        self._keep = []
        self._store_ptrs = {}
        self._fast = {}
        self._graphs = None  # pkv_step_graph cache of the repeated step, created on first use
        self.use_graph = _STEP_GRAPH
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.set_sequences(seq_ids, capacity)

    def __del__(self):
        g = getattr(self, "_graphs", None)
        if g is not None and _lib is not None:
            try:
                torch_sync = __import__("torch").cuda.synchronize
                torch_sync(self.device)  # executable graphs may still run
                self._lib.pkv_step_graph_destroy(g)
            except Exception:
                pass
            self._graphs = None

    def graph_stats(self):
        """(graph launches, graph builds) of the repeated-step CUDA graphs."""
        if self._graphs is None:
            return 0, 0
        n, b = C.c_int64(), C.c_int64()
        _lib.check(self._lib.pkv_step_graph_stats(self._graphs, C.byref(n), C.byref(b)), "pkv_step_graph_stats")
        return n.value, b.value

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
            if self._cap:  # in-flight copies may still read the old ring / host sources
                torch.cuda.current_stream(self.device).synchronize()
            self._keep_slot = [None] * 4
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
            self._bufs = {}
        self._ring_ptrs = [(h.data_ptr(), d.data_ptr(), e.cuda_event) for h, d, e in self._ring]
        self._members = object()  # invalidates the cached stage fields
        self._fast = {}
        self._slot = 0
        self._cur = None
        self._args.n_queries = self.n

    def _native_pages(self) -> bool:
        """All attached stores share one row size, so the native stage does
        the page clears / copies for every store."""
        stores = self.pool._stores
        key = [id(s) for s in stores]
        if self._stage_stores != key:
            self._uniform = len({s.row_bytes for s in stores}) == 1
            if self._uniform:
                self._kc = (C.c_void_p * len(stores))(*[s.k_cache.data_ptr() for s in stores])
                self._vc = (C.c_void_p * len(stores))(*[s.v_cache.data_ptr() for s in stores])
            self._stage_stores = key
        return self._uniform

    def _stage_setup(self):
        """Fill the stage arguments for the next ring slot; returns the slot.
        Fields that only change with the membership, the attached stores or
        the mirror tensor are rewritten only when those change."""
        if self.n == 0:
            raise ValueError("the decode batch is empty")
        slot = self._slot
        self._slot = (slot + 1) % len(self._ring)
        a = self._stage
        a.meta_host, a.meta_dev, a.slot_event = self._ring_ptrs[slot]
        native_pages = self._native_pages()
        if self._stage_fixed != (self._stage_stores, self._members):
            stores = self.pool._stores
            a.pool, a.seqs, a.n = self.pool._h, self.handles.ctypes.data, self.n
            a.page_size, a.hq, a.hkv = self.pool.page_size, self.config.head_count, self.config.kv_head_count
            a.meta_cap = self._ring[0][0].numel()
            a.n_stores = len(stores) if native_pages else 0
            a.k_caches = C.cast(self._kc, C.c_void_p) if native_pages else None
            a.v_caches = C.cast(self._vc, C.c_void_p) if native_pages else None
            a.row_bytes = stores[0].row_bytes if native_pages else 0
            self._stage_fixed = (self._stage_stores, self._members)
        mirror = self.pool._mirror
        if mirror is None or mirror.device != self.device:
            mirror = self.pool.device_table(self.device)
        if mirror is not self._stage_mirror:
            a.mirror_dev, a.mirror_rows, a.mirror_cols = mirror.data_ptr(), mirror.shape[0], mirror.shape[1]
            self._stage_mirror = mirror
        return slot

    def _stage_finish(self, slot) -> int:
        """Page work the native stage could not do (mixed row sizes) and the
        full mirror re-export after a block-table shape change."""
        a = self._stage
        launches = a.launches
        if not a.n_stores:  # stores of different row sizes: page work through the stores
            stores = self.pool._stores
            meta = self._ring[slot][0].numpy()
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

    @on_device(_self_device)
    def prepare(self, _sp=None) -> int:
        """Host work of one token step in one native call
        (pkv_decode_step_stage): allocator bookkeeping (grow, copy-on-write,
        logical_len), the packed metadata + work plan, their upload, the page
        clears / copies in every attached store and the block-table mirror
        update.  Returns the number of auxiliary kernels it launched."""
        slot = self._stage_setup()
        st = self._lib.pkv_decode_step_stage(self._stage_p, _sp if _sp is not None else _stream(self.device))
        if st:
            _lib.check(st, "pkv_decode_step_stage")
        return self._stage_finish(slot)

    def _buffer(self, name, shape, dtype):
        """Persistent device buffer (capacity-sized) for host-side inputs /
        outputs; a view of the first n rows is returned."""
        import torch

        key = (name, dtype, shape)
        view = self._bufs.get(key)
        if view is None:  # a capacity-sized buffer per (name, dtype, row shape); cached n-row view
            base = self._bufs.get((name, dtype, shape[1:], self._cap))
            if base is None:
                base = torch.empty((self._cap,) + tuple(shape[1:]), dtype=dtype, device=self.device)
                self._bufs[(name, dtype, shape[1:], self._cap)] = base
            view = self._bufs[key] = base[:shape[0]]
        return view

    def _packed(self, q_shape, kv_shape, dtype):
        """Adjacent device views q | k | v of one capacity-sized buffer, the
        layout of a packed host input (one H2D copy)."""
        import torch

        key = ("packed", q_shape, kv_shape, dtype)
        views = self._bufs.get(key)
        if views is None:
            qn, kvn = int(np.prod(q_shape)), int(np.prod(kv_shape))
            base = self._bufs.get(("packed_base", dtype, self._cap))
            per_row = (q_shape[1] + 2 * kv_shape[1]) * q_shape[2]
            if base is None:
                base = torch.empty(self._cap * per_row, dtype=dtype, device=self.device)
                self._bufs[("packed_base", dtype, self._cap)] = base
            views = (base[:qn].view(q_shape), base[qn:qn + kvn].view(kv_shape),
                     base[qn + kvn:qn + 2 * kvn].view(kv_shape))
            self._bufs[key] = views
        return views

    @staticmethod
    def _one_allocation(*tensors) -> bool:
        """Adjacent host tensors are one copy only if they share a storage
        (separately pinned buffers may sit back to back by chance)."""
        base = tensors[0].untyped_storage().data_ptr()
        return all(t.untyped_storage().data_ptr() == base for t in tensors[1:])

    @staticmethod
    def packed_host_inputs(n, hq, hkv, d, dtype, pin=True):
        """Host buffers for step(): q [n,Hq,D], k_new / v_new [n,Hkv,D] as
        adjacent views of one (pinned) allocation, so the step moves them
        with a single host-to-device copy."""
        import torch

        base = torch.empty(n * (hq + 2 * hkv) * d, dtype=dtype)
        if pin:
            base = base.pin_memory()
        qn, kvn = n * hq * d, n * hkv * d
        return (base[:qn].view(n, hq, d), base[qn:qn + kvn].view(n, hkv, d),
                base[qn + kvn:qn + 2 * kvn].view(n, hkv, d))

    def _input(self, x, dtype, shape, name, zero_copy=False):
        """-> (device tensor, host pointer or None, bytes).  CPU inputs are
        copied by the native step into a persistent device buffer (pin them
        for an asynchronous copy); device inputs are used in place.  Records
        in self._direct whether the caller's own buffer is used (no
        conversion copy), which makes the call repeatable by _step_fast."""
        import torch

        if type(x) is torch.Tensor and x.dtype is dtype and not x.is_cuda and x.shape == shape \
                and x.is_contiguous():  # fast path: a host tensor ready to copy
            self._keep.append(x)
            self._direct.append(True)
            if (_ZERO_COPY_IN or zero_copy) and x.is_pinned():
                return x, None, 0  # the kernel reads the mapped host rows itself
            return self._buffer(name, shape, dtype), x.data_ptr(), x.nbytes
        self._direct.append(False)
        if not isinstance(x, torch.Tensor):
            x = torch.from_numpy(np.ascontiguousarray(x))
        if tuple(x.shape) != shape:
            raise ShapeMismatch(f"{name} has shape {tuple(x.shape)}, expected {shape}")
        if x.device.type == "cpu":
            if x.dtype != dtype or not x.is_contiguous():
                x = x.to(dtype).contiguous()
            self._keep.append(x)
            return self._buffer(name, shape, dtype), x.data_ptr(), x.numel() * x.element_size()
        if x.device != self.device or x.dtype != dtype or not x.is_contiguous():
            x = x.to(device=self.device, dtype=dtype, non_blocking=True).contiguous()
            return x, None, 0
        self._direct[-1] = True
        return x, None, 0

    def step(self, queries, k_new, v_new, *, out=None, out_dtype=None, layer: int = 0, advance: bool = True,
             precision: str = "auto"):
        """Append one token per sequence into `stores[layer]` and attend.

        queries [B, Hq, D]; k_new / v_new [B, Hkv, D] (numpy or torch, any
        device).  With `advance` (the default) the whole step — copies of CPU
        inputs, allocator + plan + metadata upload, page work, the fused
        append + decode launch and the copy into a CPU `out` — is ONE native
        call (pkv_decode_step).  `out` (optional) is a [B, Hq, D] tensor the
        result is written to: on the device, or on the host (pinned: the
        copy is asynchronous on the current stream, synchronise before
        reading it, as with a non_blocking torch copy).

        A serving loop calls this with the same input / output buffers every
        token; such a repeated call (same tensor objects, same storage) skips
        the argument checks and marshalling and re-uses the argument blocks
        prepared by the first call (`_FastStep`)."""
        if out is not None and advance:
            e = self._fast.get((id(queries), id(k_new), id(v_new), id(out), layer, precision))
            if e is not None and e.valid(self, queries, k_new, v_new, out):
                return self._step_fast(e)
        return self._step_full(queries, k_new, v_new, out=out, out_dtype=out_dtype, layer=layer,
                               advance=advance, precision=precision)

    def _step_fast(self, e):
        import torch

        if torch.cuda.current_device() != self._dev_index:
            with torch.cuda.device(self.device):
                return self._step_fast(e)
        sp = torch._C._cuda_getCurrentRawStream(self._dev_index)
        slot = self._slot
        self._slot = (slot + 1) % len(self._ring)
        st_args = self._stage
        st_args.meta_host, st_args.meta_dev, st_args.slot_event = self._ring_ptrs[slot]
        mirror = self.pool._mirror
        if mirror is not self._stage_mirror:  # re-exported mirror: refresh the table fields
            self._stage_setup_mirror()
        if e.mirror is not self._stage_mirror:
            e.args.block_table, e.args.bt_stride = st_args.mirror_dev, st_args.mirror_cols
            e.mirror = self._stage_mirror
        if e.graph_ok and self.use_graph:
            if self._graphs is None:
                h = C.c_void_p()
                _lib.check(self._lib.pkv_step_graph_create(C.byref(h)), "pkv_step_graph_create")
                self._graphs = h
            st = self._lib.pkv_decode_step_graph(self._graphs, self._stage_p, e.args_p, e.io_p, C.c_void_p(sp))
        else:
            st = self._lib.pkv_decode_step(self._stage_p, e.args_p, e.io_p, C.c_void_p(sp))
        if st:
            _lib.check(st, "pkv_decode_step")
        self._cur = slot
        self._used.value = st_args.meta_used
        if st_args.needs_resync or not e.io.launched:  # block-table shape change: the general path
            self._stage_finish_resync(e, sp)
        else:
            self.last_launches = e.io.launches
        return e.result

    def _stage_setup_mirror(self):
        a = self._stage
        mirror = self.pool._mirror
        if mirror is None or mirror.device != self.device:
            mirror = self.pool.device_table(self.device)
        if mirror is not self._stage_mirror:
            a.mirror_dev, a.mirror_rows, a.mirror_cols = mirror.data_ptr(), mirror.shape[0], mirror.shape[1]
            self._stage_mirror = mirror

    def _stage_finish_resync(self, e, sp):
        """Fast-path tail after a block-table shape change: full mirror
        re-export, then the attention launch on it (as in _step_full)."""
        if self._stage.needs_resync:
            self.pool.device_table(self.device)
        launches = self._stage.launches
        if not e.io.launched:
            mirror = self.pool.device_table(self.device)
            e.args.block_table, e.args.bt_stride = mirror.data_ptr(), mirror.shape[1]
            e.mirror = None
            st = self._lib.pkv_paged_attention(e.args_p, C.c_void_p(sp))
            if st:
                _lib.check(st, "pkv_paged_attention")
            if e.out_host is not None:
                e.out_host.copy_(e.out_dev, non_blocking=True)
            launches += 1 if e.tensor else 4
        else:
            launches = e.io.launches
        self.last_launches = launches

    @on_device(_self_device)
    def _step_full(self, queries, k_new, v_new, *, out=None, out_dtype=None, layer: int = 0, advance: bool = True,
                   precision: str = "auto"):
        """Append one token per sequence into `stores[layer]` and attend.

        queries [B, Hq, D]; k_new / v_new [B, Hkv, D] (numpy or torch, any
        device).  With `advance` (the default) the whole step — copies of CPU
        inputs, allocator + plan + metadata upload, page work, the fused
        append + decode launch and the copy into a CPU `out` — is ONE native
        call (pkv_decode_step).  `out` (optional) is a [B, Hq, D] tensor the
        result is written to: on the device, or on the host (pinned: the
        copy is asynchronous on the current stream, synchronise before
        reading it, as with a non_blocking torch copy)."""
        import torch

        sp = _stream(self.device)
        if not advance or not self._native_pages():
            return self._step_split(queries, k_new, v_new, out=out, out_dtype=out_dtype, layer=layer,
                                    advance=advance, precision=precision, sp=sp)
        fast_key = (id(queries), id(k_new), id(v_new), id(out), layer, precision) if out is not None else None
        store: KvStore = self.stores[layer]
        cfg = self.config
        n = self.n
        self._keep = []
        self._direct = []
        qd = queries.dtype if isinstance(queries, torch.Tensor) else None
        q_t = qd if qd in self._qcodes else torch.float32
        q, q_host, q_bytes = self._input(queries, q_t, (n, cfg.head_count, cfg.head_dim), "queries")
        kv_shape = (n, cfg.kv_head_count, cfg.head_dim)
        k, k_host, kv_bytes = self._input(k_new, store.torch_dtype, kv_shape, "k_new", _ZERO_COPY_KV)
        v, v_host, _ = self._input(v_new, store.torch_dtype, kv_shape, "v_new", _ZERO_COPY_KV)
        if q_host and k_host == q_host + q_bytes and v_host == k_host + kv_bytes and q_t is store.torch_dtype \
                and self._one_allocation(queries, k_new, v_new):
            # q | k | v adjacent in one host buffer (a fused QKV projection's
            # output, planar): ONE host-to-device copy into a packed buffer
            q, k, v = self._packed(q.shape, k.shape, q_t)
            q_bytes, k_host, v_host = q_bytes + 2 * kv_bytes, None, None
        out_host = None
        if out is None:
            out_t, out_code = (torch.float32, _lib.PKV_F32) if out_dtype is None else torch_dtype(out_dtype)
            o = torch.empty((n, cfg.head_count, cfg.head_dim), dtype=out_t, device=self.device)
            result = o
        else:
            if tuple(out.shape) != (n, cfg.head_count, cfg.head_dim) or not out.is_contiguous() \
                    or out.dtype not in self._qcodes:
                raise ShapeMismatch("out must be a contiguous [B, Hq, D] float32/float16/bfloat16 tensor")
            out_code = self._qcodes[out.dtype]
            if out.device.type == "cpu" and _ZERO_COPY_OUT and out.is_pinned():
                o = out  # the kernel stores straight into mapped pinned memory
            elif out.device.type == "cpu":
                o = self._buffer("out", tuple(out.shape), out.dtype)
                out_host = out
            else:
                o = out
            result = out
        slot = self._stage_setup()
        ptrs = self._store_ptrs.get(id(store))
        if ptrs is None:
            ptrs = (store.k_cache.data_ptr(), store.v_cache.data_ptr(), store.dtype_code, store.page_size)
            self._store_ptrs[id(store)] = ptrs
        a = self._args
        a.q, a.q_dtype = q.data_ptr(), self._qcodes[q.dtype]
        a.k_cache, a.v_cache, a.kv_dtype, a.page_size = ptrs
        a.block_table, a.bt_stride = self._stage.mirror_dev, self._stage.mirror_cols
        a.out, a.out_dtype = o.data_ptr(), out_code
        a.mode = PRECISION_MODES[precision]
        a.k_new, a.v_new = k.data_ptr(), v.data_ptr()
        io = self._io
        io.q_host, io.k_host, io.v_host = q_host, k_host, v_host
        io.q_bytes, io.kv_bytes = q_bytes, kv_bytes
        io.out_host = out_host.data_ptr() if out_host is not None else None
        io.out_bytes = out_host.numel() * out_host.element_size() if out_host is not None else 0
        st = self._lib.pkv_decode_step(self._stage_p, self._args_p, self._io_p, sp)
        # host sources stay referenced until this slot's event (recorded after
        # their copies) has been waited on by the call that reuses the slot
        self._keep_slot[slot] = self._keep
        if st:
            _lib.check(st, "pkv_decode_step")
        launches = self._stage_finish(slot)
        if not io.launched:  # block-table shape changed: launch on the re-exported mirror
            mirror = self.pool.device_table(self.device)
            a.block_table, a.bt_stride = mirror.data_ptr(), mirror.shape[1]
            st = self._lib.pkv_paged_attention(self._args_p, sp)
            if st:
                _lib.check(st, "pkv_paged_attention")
            if out_host is not None:
                out_host.copy_(o, non_blocking=True)
            tensor = (store.dtype_code == _lib.PKV_BF16 and precision != "exact") or precision == "tensor"
            launches += 1 if tensor else 4
        else:
            launches = io.launches
        self.last_launches = launches
        if fast_key is not None and all(type(x) is torch.Tensor for x in (queries, k_new, v_new)):
            # every buffer used in place (host pointer or device tensor of the
            # caller's own objects): later calls with these objects skip to
            # _step_fast with a private copy of the argument blocks
            if all(self._direct) and (o is out or out_host is out):
                tensor = (store.dtype_code == _lib.PKV_BF16 and precision != "exact") or precision == "tensor"
                if len(self._fast) >= 16:
                    self._fast.clear()
                self._fast[fast_key] = _FastStep(self, (queries, k_new, v_new, out), result, out_host, o,
                                                 tensor)
        return result

    def _step_split(self, queries, k_new, v_new, *, out, out_dtype, layer, advance, precision, sp):
        """prepare() (when advancing) + the attention launch as two calls:
        the multi-layer form (advance=False) and stores of mixed row sizes."""
        import torch

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
        host_out = None
        if out is not None and out.device.type == "cpu":
            host_out, out = out, None
            out_dtype = host_out.dtype
        if out is None:
            out_t, out_code = (torch.float32, _lib.PKV_F32) if out_dtype is None else torch_dtype(out_dtype)
            out = torch.empty((n, cfg.head_count, cfg.head_dim), dtype=out_t, device=self.device)
        else:
            if tuple(out.shape) != (n, cfg.head_count, cfg.head_dim) or not out.is_contiguous() \
                    or out.dtype not in self._qcodes:
                raise ShapeMismatch("out must be a contiguous [B, Hq, D] float32/float16/bfloat16 tensor")
            out_code = self._qcodes[out.dtype]
        md = dev.data_ptr()
        hp = host.data_ptr()
        ptrs = self._store_ptrs.get(id(store))
        if ptrs is None:
            ptrs = (store.k_cache.data_ptr(), store.v_cache.data_ptr(), store.dtype_code, store.page_size)
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
        if host_out is not None:
            host_out.copy_(out, non_blocking=True)
            return host_out
        return out
