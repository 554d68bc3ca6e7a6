"""Attention entry points — drop-in for reference attention.py:26-378.

`paged_attention(queries, store, meta, config)` keeps the reference signature
(attention.py:332-354) and runs on the device:

* decode-shaped and general metas -> K2 split-K flash decode + K2c combine
  (csrc/kernels.cu), fp32/fp16/bf16 caches;
* bf16 suffix / self-attention metas with long query runs -> K3 tcgen05
  prefill (csrc/prefill_sm100.cu) when the shape is supported.

The reference mask predicate (attention.py:113-134) admits, for query i of
sequence s, exactly the key prefix [0, n_i) of s with n_i = min(q_pos+1, len)
when causal and len otherwise; the host reduces every MaskMeta to that count,
so kernels never see the block mask.  `block_mask` / `skip_empty` are accepted
for signature compatibility: the reference guarantees skip == no-skip bitwise
(test_attention.py:206-210), and the device path only ever visits allowed keys.
Grouped-query attention (not in the reference) is enabled by
`AttentionConfig.kv_head_count`; q head h reads kv head h // G.
"""

from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _lib
from .errors import ConfigError, NoAllowedKeys, OutOfRange, ShapeMismatch
from .store import BatchView, KvStore, _ptr, _stream, on_device, stage_upload, to_device, torch_dtype


class BlockKind(IntEnum):
    EMPTY = 0
    PARTIAL = 1
    FULL = 2


@dataclass
class AttentionConfig:
    """attention.py:32-48, plus `kv_head_count` for grouped-query attention."""

    head_count: int
    head_dim: int
    scale: float | None = None
    causal: bool = True
    page_size: int = 64
    kv_head_count: int | None = None

    def __post_init__(self):
        if self.head_count <= 0 or self.head_dim <= 0:
            raise ValueError("head_count and head_dim must be positive")
        if self.page_size <= 0 or self.page_size & (self.page_size - 1):
            raise ValueError("page_size must be a positive power of two")
        if self.scale is None:
            self.scale = 1.0 / math.sqrt(self.head_dim)
        if self.scale <= 0:
            raise ValueError("scale must be positive")
        if self.kv_head_count is None:
            self.kv_head_count = self.head_count
        if self.kv_head_count <= 0 or self.head_count % self.kv_head_count:
            raise ValueError("head_count must be a multiple of kv_head_count")


@dataclass
class MaskMeta:
    """Query-side addressing against a KV batch view (attention.py:51-110)."""

    view: BatchView
    q_seq: np.ndarray
    q_pos: np.ndarray

    def __post_init__(self):
        self.q_seq = np.asarray(self.q_seq, dtype=np.int64)
        self.q_pos = np.asarray(self.q_pos, dtype=np.int64)
        if self.q_seq.shape != self.q_pos.shape or self.q_seq.ndim != 1:
            raise ShapeMismatch("q_seq and q_pos must be 1-D vectors of equal length")
        if self.q_seq.size:
            if (np.diff(self.q_seq) < 0).any():
                raise ValueError("q_seq must be non-decreasing (sequence-major order)")
            if self.q_seq.min() < 0 or self.q_seq.max() >= len(self.view.lengths):
                raise OutOfRange("q_seq refers to a sequence outside the view")
            if (self.q_pos < 0).any() or (self.q_pos >= self.view.lengths[self.q_seq]).any():
                raise OutOfRange("query positions must be < their sequence length")

    @property
    def query_count(self) -> int:
        return int(self.q_seq.shape[0])

    @classmethod
    def self_attention(cls, view: BatchView) -> "MaskMeta":
        return cls(view=view, q_seq=view.slot_seq.copy(), q_pos=view.slot_local.copy())._sealed()

    def _sealed(self) -> "MaskMeta":
        """Mark the constructor's own (fresh) query arrays read-only: a meta
        built by self_attention / decode / suffix can then be recognised as
        unchanged by identity (the prefill fast path of paged_attention)."""
        self.q_seq.flags.writeable = False
        self.q_pos.flags.writeable = False
        return self

    @classmethod
    def decode(cls, view: BatchView) -> "MaskMeta":
        n = len(view.lengths)
        if (view.lengths <= 0).any():
            raise OutOfRange("decode meta requires every sequence to have length >= 1")
        return cls(view=view, q_seq=np.arange(n, dtype=np.int64), q_pos=view.lengths - 1)._sealed()

    @classmethod
    def suffix(cls, view: BatchView, q_lengths) -> "MaskMeta":
        q_lengths = np.asarray(q_lengths, dtype=np.int64)
        if q_lengths.shape != view.lengths.shape:
            raise ShapeMismatch("one query count per sequence required")
        if (q_lengths < 0).any() or (q_lengths > view.lengths).any():
            raise OutOfRange("query counts must be within sequence lengths")
        q_seq = np.repeat(np.arange(len(q_lengths), dtype=np.int64), q_lengths)
        if q_lengths.sum():
            q_pos = np.concatenate([np.arange(n - q, n, dtype=np.int64)
                                    for n, q in zip(view.lengths, q_lengths)])
        else:
            q_pos = np.zeros(0, dtype=np.int64)
        return cls(view=view, q_seq=q_seq, q_pos=q_pos)._sealed()


def mask_allow(q_index: int, k_index: int, meta: MaskMeta, causal: bool = True) -> bool:
    """Pointwise predicate over flat indices (attention.py:113-134)."""
    if q_index < 0 or q_index >= meta.query_count:
        raise OutOfRange(f"query index {q_index} outside flat query batch")
    view = meta.view
    if k_index < 0 or k_index >= view.total_slots:
        raise OutOfRange(f"kv index {k_index} outside flat batch of {view.total_slots}")
    q_seq = int(meta.q_seq[q_index])
    k_seq = int(view.slot_seq[k_index])
    if q_seq != k_seq:
        return False
    k_local = int(view.slot_local[k_index])
    if k_local >= int(view.lengths[k_seq]):
        return False
    return not (causal and k_local > int(meta.q_pos[q_index]))


def allowed_key_counts(meta: MaskMeta, causal: bool) -> np.ndarray:
    """Length of the allowed key prefix of every query (see module doc)."""
    lens = meta.view.lengths[meta.q_seq]
    return np.minimum(meta.q_pos + 1, lens) if causal else lens.copy()


@dataclass
class BlockMask:
    """FULL/PARTIAL/EMPTY per (query tile, kv tile) of the flat view
    (attention.py:137-168); host metadata used for KernelStats parity."""

    kinds: np.ndarray = field(repr=False)
    page_size: int
    q_len: int
    kv_len: int

    def kind(self, q_block: int, k_block: int) -> BlockKind:
        return BlockKind(int(self.kinds[q_block, k_block]))

    def counts(self) -> dict:
        return {"empty": int((self.kinds == 0).sum()), "partial": int((self.kinds == 1).sum()),
                "full": int((self.kinds == 2).sum())}


def build_block_mask(meta: MaskMeta, config: AttentionConfig) -> BlockMask:
    """Tile classification (attention.py:171-210), vectorised per query tile:
    query i admits the flat key interval [prefix[s], prefix[s] + n_i)."""
    bs = config.page_size
    nq, nk = meta.query_count, meta.view.total_slots
    n_qb, n_kb = -(-nq // bs), -(-nk // bs)
    kinds = np.zeros((n_qb, n_kb), dtype=np.int8)
    if n_qb and n_kb:
        lo = meta.view.prefix_sums[meta.q_seq]
        hi = lo + allowed_key_counts(meta, config.causal)
        k0 = np.arange(n_kb) * bs
        k1 = np.minimum(k0 + bs, nk)
        for qb in range(n_qb):
            a = lo[qb * bs:(qb + 1) * bs, None]
            b = hi[qb * bs:(qb + 1) * bs, None]
            hit = ((a < k1[None]) & (b > k0[None])).any(axis=0)
            full = ((a <= k0[None]) & (b >= k1[None])).all(axis=0)
            kinds[qb] = np.where(full, 2, np.where(hit, 1, 0))
    return BlockMask(kinds=kinds, page_size=bs, q_len=nq, kv_len=nk)


@dataclass
class KernelStats:
    """Per-run instrumentation (attention.py:213-226), computed on the host
    from the metadata: the device kernels never visit disallowed keys."""

    visited_blocks: int = 0
    skipped_blocks: int = 0
    allowed_pairs: int = 0
    head_count: int = 0
    head_dim: int = 0

    @property
    def attention_flops(self) -> int:
        return 4 * self.head_count * self.head_dim * self.allowed_pairs


def _fill_stats(stats: KernelStats, meta: MaskMeta, config: AttentionConfig, nkeys, block_mask):
    stats.head_count, stats.head_dim = config.head_count, config.head_dim
    if meta.query_count == 0:
        return
    bm = block_mask if block_mask is not None else build_block_mask(meta, config)
    visited = int((bm.kinds != 0).sum())
    stats.visited_blocks += visited
    stats.skipped_blocks += int(bm.kinds.size) - visited
    stats.allowed_pairs += int(nkeys.sum())


def _check_queries(queries, meta: MaskMeta, config: AttentionConfig):
    expected = (meta.query_count, config.head_count, config.head_dim)
    shape = tuple(queries.shape) if hasattr(queries, "shape") else np.asarray(queries).shape
    if shape != expected:
        raise ShapeMismatch(f"expected queries of shape {expected}, got {shape}")


class _Workspace:
    """Scratch for split partials (and the CUDA-core device plan), one buffer
    per (device, stream): launches on one stream are ordered, so they may
    share it; concurrent streams must not."""

    _bufs: dict = {}

    @classmethod
    def get(cls, device, nbytes: int):
        import torch

        key = (device, torch.cuda.current_stream(device).cuda_stream)
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            cls._bufs[key] = buf
        return buf


def _q_tensor(queries, device):
    import torch

    q = queries if isinstance(queries, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(queries))
    if q.dtype == torch.float64:
        q = q.float()
    q = q.to(device).contiguous()
    _, code = torch_dtype(q.dtype)
    return q, code


PRECISION_MODES = {"auto": 0, "exact": 1, "tensor": 2, "prefill": 2}


@on_device(lambda *a, **k: k.get("device"))
def _launch_attention(q, qcode, meta, config, nkeys, *, k, v, kv_code, bt, bt_stride, seq_row,
                      seq_start, out_dtype, device, precision="auto"):
    import torch

    nq = meta.query_count
    out_t, out_code = torch_dtype(out_dtype)
    out = torch.empty((nq, config.head_count, config.head_dim), dtype=out_t, device=device)
    if nq == 0:
        return out
    # one packed upload: [q_seq | q_nkeys | seq_row (or seq_start as int64) | plan]
    q_seq = meta.q_seq.astype(np.int32)
    rows_by_seq = seq_row if bt is not None else seq_start
    q_row = np.asarray(rows_by_seq, dtype=np.int64)[meta.q_seq]
    if q_row.size and (q_row.max() >= 2 ** 31):
        raise OutOfRange("K/V rows beyond 2^31 are not addressable")
    plan = _lib.attention_plan(nkeys, q_row, config.page_size, config.head_count,
                               config.kv_head_count, head_dim=config.head_dim)
    seq_part = (np.asarray(seq_row, dtype=np.int32) if bt is not None
                else np.asarray(seq_start, dtype=np.int64).view(np.int32))
    nseq = seq_part.size
    # 2*nq int32 precede seq_part, so an int64 seq_start stays 8-byte aligned
    host = np.concatenate([q_seq, nkeys.astype(np.int32), seq_part, plan])
    dev = stage_upload(device, host)
    base = dev.data_ptr()
    seq_ptr = base + 4 * (2 * nq)
    plan_ptr = seq_ptr + 4 * nseq
    ws_bytes = _lib.load().pkv_attention_workspace_bytes(nq, config.head_count, config.head_dim)
    ws = _Workspace.get(device, ws_bytes)
    args = _lib.AttentionArgs(
        q=q.data_ptr(), q_dtype=qcode, n_queries=nq, q_seq=base, q_nkeys=base + 4 * nq,
        k_cache=k.data_ptr(), v_cache=v.data_ptr(), kv_dtype=kv_code,
        block_table=bt.data_ptr() if bt is not None else None, bt_stride=bt_stride,
        seq_row=seq_ptr if bt is not None else None, seq_start=seq_ptr if bt is None else None,
        page_size=config.page_size, hq=config.head_count, hkv=config.kv_head_count,
        head_dim=config.head_dim, scale=float(config.scale), out=out.data_ptr(), out_dtype=out_code,
        workspace=ws.data_ptr(), workspace_bytes=ws.numel(), num_sms=0, target_waves=0,
        mode=PRECISION_MODES[precision], plan=plan_ptr, plan_host=plan.ctypes.data)
    _lib.check(_lib.load().pkv_paged_attention(C.byref(args), _stream(device)), "pkv_paged_attention")
    return out


PREFILL_MIN_RUN = 16  # longest per-sequence query run that makes the K3 tile worthwhile


def suffix_runs(meta: MaskMeta):
    """(q_start, q_len) per view sequence when the queries of every sequence
    are one run of consecutive positions ending at its last key — the shape
    of MaskMeta.self_attention / .suffix (attention.py:81-84, 98-110) that K3
    executes — else None."""
    n_seq = len(meta.view.lengths)
    q_len = np.bincount(meta.q_seq, minlength=n_seq).astype(np.int64)
    q_start = np.zeros(n_seq, dtype=np.int64)
    if n_seq > 1:
        q_start[1:] = np.cumsum(q_len)[:-1]
    if meta.query_count == 0:
        return q_start, q_len
    lens = meta.view.lengths.astype(np.int64)
    first = lens - q_len
    idx = np.arange(meta.query_count, dtype=np.int64)
    want = first[meta.q_seq] + idx - q_start[meta.q_seq]
    if not np.array_equal(want, meta.q_pos):
        return None
    return q_start, q_len


@dataclass
class _PrefillRoute:
    """The K3 route of one call: the memoised plan (host view), its size and
    the generation naming it (pkv_prefill_plan_meta)."""

    plan: np.ndarray
    n_items: int
    generation: int


_plan_tls = threading.local()


def _prefill_plan_meta(meta: MaskMeta, config: AttentionConfig, rows, min_run: int):
    """(n_items, longest run, plan view, generation): -1 items when the meta
    is not suffix-shaped; 0 items when no run reaches `min_run`.  One native
    pass (suffix check, run lengths, memoised planner)."""
    view = meta.view
    n_seq, nq = len(view.lengths), meta.query_count
    qt = 128 // (config.head_count // config.kv_head_count)
    cap = config.kv_head_count * (nq // (2 * qt) + n_seq + 1) * _lib.PREFILL_ITEM_INTS
    buf = getattr(_plan_tls, "buf", None)
    if buf is None or buf.size < cap:
        buf = _plan_tls.buf = np.empty(max(cap, 1 << 14), dtype=np.int32)
        _plan_tls.out = np.zeros(3, dtype=np.int64)
    out = _plan_tls.out
    q_seq = np.ascontiguousarray(meta.q_seq, dtype=np.int64)
    q_pos = np.ascontiguousarray(meta.q_pos, dtype=np.int64)
    lens = np.ascontiguousarray(view.lengths, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    base = out.ctypes.data
    _lib.check(_lib.load().pkv_prefill_plan_meta(
        q_seq.ctypes.data, q_pos.ctypes.data, nq, lens.ctypes.data, rows.ctypes.data, n_seq,
        config.head_count, config.kv_head_count, int(bool(config.causal)), min_run, buf.ctypes.data, buf.size,
        base, base + 8, base + 16), "pkv_prefill_plan_meta")
    n_items, max_run, gen = (int(x) for x in out)
    return n_items, max_run, buf[: max(n_items, 0) * _lib.PREFILL_ITEM_INTS], gen


def _prefill_route(meta, config, kv_code, precision, rows):
    """The K3 plan, or None to use K2.  "auto" sends bf16 caches with
    query runs of >= PREFILL_MIN_RUN positions (fp16 stays on the fp32
    CUDA-core kernel and its 1e-5 contract, like the decode dispatch);
    "tensor" also takes fp16; "prefill" forces K3 for any suffix-shaped meta
    (attention.py:81-84, 98-110).  `rows`: mirror row (paged) or first K/V
    row (gathered) per view sequence."""
    if precision == "exact":
        return None
    if precision == "auto" and kv_code != _lib.PKV_BF16 or kv_code not in (_lib.PKV_BF16, _lib.PKV_F16):
        return None
    supported = _lib.load().pkv_prefill_supported(config.head_count, config.kv_head_count, config.head_dim,
                                                  config.page_size, kv_code)
    if not supported:
        if precision == "prefill":
            raise ConfigError("the tcgen05 prefill needs a suffix-shaped meta over a 16-bit cache with "
                              "head_dim 64/128, page_size >= 8 and 128 % (hq/hkv) == 0")
        return None
    rows = np.asarray(rows)
    if rows.size and rows.max() >= 2 ** 31:
        raise OutOfRange("K/V rows beyond 2^31 are not addressable")
    min_run = 1 if precision == "prefill" else PREFILL_MIN_RUN
    n_items, max_run, plan, gen = _prefill_plan_meta(meta, config, rows, min_run)
    if n_items < 0:
        if precision == "prefill":
            raise ConfigError("the tcgen05 prefill needs a suffix-shaped meta over a 16-bit cache with "
                              "head_dim 64/128, page_size >= 8 and 128 % (hq/hkv) == 0")
        return None
    if max_run < min_run or meta.query_count == 0:
        return None if precision != "prefill" else _PrefillRoute(plan, 0, gen)
    return _PrefillRoute(plan.reshape(-1, _lib.PREFILL_ITEM_INTS), n_items, gen)


# device copy of the last K3 plan per (host thread, device, stream): a call
# whose memoised plan has the same generation reuses it (layers of a model)
_prefill_dev_plans: dict = {}


def _device_plan(route: _PrefillRoute, device):
    import torch

    key = (threading.get_ident(), device, _stream(device).value or 0)  # legacy default stream: 0
    ent = _prefill_dev_plans.get(key)
    size = route.n_items * _lib.PREFILL_ITEM_INTS
    if ent is not None and ent[0] == route.generation and ent[2] == size:
        return ent[1]
    staged = stage_upload(device, route.plan.reshape(-1))
    dev = ent[1] if ent is not None and ent[1].numel() >= size else torch.empty(
        max(size, 1 << 12), dtype=torch.int32, device=device)
    dev[:size].copy_(staged)  # stream-ordered behind any kernel still reading the old plan
    _prefill_dev_plans[key] = (route.generation, dev, size)
    return dev


@on_device(lambda *a, **k: k.get("device"))
def _launch_prefill(q, meta, config, runs, *, k, v, kv_code, bt, rows, out_dtype, device, prof=None,
                    route: _PrefillRoute | None = None, memo: dict | None = None):
    """K3: one tcgen05 launch over every sequence's query run.  Paged mode:
    `bt` is the device block-table mirror and `rows` the mirror row of each
    view sequence; gathered mode (bt None): `rows` is each sequence's first
    row in the contiguous K/V."""
    import torch

    nq = meta.query_count
    out_t, out_code = torch_dtype(out_dtype)
    if out_code not in (_lib.PKV_F32, kv_code):
        out_t, out_code = torch.float32, _lib.PKV_F32
    out = torch.empty((nq, config.head_count, config.head_dim), dtype=out_t, device=device)
    if nq == 0:
        return out
    q = q.to(k.dtype).contiguous()
    if route is not None:
        plan, dev_plan = route.plan, _device_plan(route, device)
    else:  # explicit runs (tools): plan and upload here
        rows = np.asarray(rows, dtype=np.int64)
        if rows.size and rows.max() >= 2 ** 31:
            raise OutOfRange("K/V rows beyond 2^31 are not addressable")
        q_start, q_len = runs
        plan = _lib.prefill_plan(q_start, q_len, meta.view.lengths, rows, config.head_count,
                                 config.kv_head_count, config.causal)
        dev_plan = stage_upload(device, plan.reshape(-1))
    args = _lib.PrefillArgs(
        q=q.data_ptr(), total_q=nq, k_cache=k.data_ptr(), v_cache=v.data_ptr(),
        kv_dtype=kv_code, cache_rows=k.shape[0], block_table=bt.data_ptr() if bt is not None else None,
        bt_stride=bt.shape[1] if bt is not None else 0, page_size=config.page_size,
        hq=config.head_count, hkv=config.kv_head_count, head_dim=config.head_dim,
        scale=float(config.scale), causal=int(bool(config.causal)), out=out.data_ptr(),
        out_dtype=out_code, plan=dev_plan.data_ptr(), n_items=plan.shape[0],
        prof_start=prof[0] if prof else None, prof_stop=prof[1] if prof else None)
    stream = _stream(device)
    _lib.check(_lib.load().pkv_paged_prefill(C.byref(args), stream), "pkv_paged_prefill")
    if memo is not None and route is not None and prof is None:
        sid = stream.value or 0
        memo.update(args=args, out=out, stream=sid,
                    plan_entry=_prefill_dev_plans.get((threading.get_ident(), device, sid)))
    return out


class _PrefillMemo:
    """The last K3 call of this host thread through paged_attention: the same
    meta / store / config again (a model's layers over one prompt batch) with
    the pool unchanged since (pkv_pool_generation) and this thread's device
    plan still in place skips the table lookups, the route and the plan, and
    relaunches the prepared argument block with the new q / out pointers."""

    __slots__ = ("meta", "view", "q_seq", "q_pos", "lengths", "ids", "store", "config", "cfg", "precision",
                 "out_dtype", "q_dtype", "q_shape", "device", "gen", "gen_buf", "gen_addr", "mirror", "args",
                 "args_ref", "stream", "plan_key", "plan_entry", "out_shape", "out_t")


_prefill_tls = threading.local()


def _cfg_key(config: AttentionConfig):
    return (config.head_count, config.head_dim, config.scale, config.causal, config.page_size,
            config.kv_head_count)


def _prefill_fast(queries, store, meta, config, out_dtype, precision):
    """paged_attention's repeat-call path (see _PrefillMemo), or None."""
    import torch

    ent = getattr(_prefill_tls, "memo", None)
    if (ent is None or ent.meta is not meta or ent.store is not store or ent.config is not config
            or ent.precision != precision or ent.out_dtype is not out_dtype):
        return None
    view = meta.view
    if (view is not ent.view or meta.q_seq is not ent.q_seq or meta.q_pos is not ent.q_pos
            or view.lengths.tobytes() != ent.lengths or view.ids != ent.ids or _cfg_key(config) != ent.cfg):
        return None
    if (not isinstance(queries, torch.Tensor) or queries.dtype != ent.q_dtype or queries.shape != ent.q_shape
            or queries.device != ent.device or not queries.is_contiguous()):
        return None
    lib = _lib.load()
    if lib.pkv_pool_generation(store.pool._h, ent.gen_addr) or ent.gen_buf.value != ent.gen:
        return None  # a table, page or mirror changed: the full path re-derives everything
    if store.pool._mirror is not ent.mirror:
        return None
    stream = torch._C._cuda_getCurrentRawStream(ent.device.index)
    if stream != ent.stream or _prefill_dev_plans.get(ent.plan_key) is not ent.plan_entry:
        return None  # another stream, or another plan was uploaded into this thread's buffer
    out = torch.empty(ent.out_shape, dtype=ent.out_t, device=ent.device)
    args = ent.args
    args.q = queries.data_ptr()
    args.out = out.data_ptr()
    _lib.check(lib.pkv_paged_prefill(ent.args_ref, C.c_void_p(stream)), "pkv_paged_prefill")
    return out


def _remember_prefill(queries, store, meta, config, out_dtype, precision, gen, rec):
    import torch

    if rec.get("plan_entry") is None or not isinstance(queries, torch.Tensor):
        return
    if (meta.q_seq.flags.writeable or meta.q_pos.flags.writeable or queries.dtype != store.k_cache.dtype
            or not queries.is_contiguous() or queries.device != store.device or store.device.index is None):
        return  # only sealed metas (MaskMeta constructors) and ready device queries repeat cheaply
    ent = _PrefillMemo()
    view = meta.view
    ent.meta, ent.view, ent.q_seq, ent.q_pos = meta, view, meta.q_seq, meta.q_pos
    ent.lengths, ent.ids = view.lengths.tobytes(), list(view.ids)
    ent.store, ent.config, ent.cfg = store, config, _cfg_key(config)
    ent.precision, ent.out_dtype = precision, out_dtype
    ent.q_dtype, ent.q_shape, ent.device = queries.dtype, queries.shape, store.device
    ent.gen = gen
    ent.gen_buf = C.c_uint64()
    ent.gen_addr = C.addressof(ent.gen_buf)
    ent.mirror = store.pool._mirror
    ent.args = rec["args"]
    ent.args_ref = C.byref(ent.args)
    ent.stream = rec["stream"]
    ent.plan_key = (threading.get_ident(), store.device, rec["stream"])
    ent.plan_entry = rec["plan_entry"]
    ent.out_shape, ent.out_t = tuple(rec["out"].shape), rec["out"].dtype
    _prefill_tls.memo = ent


def _pool_generation(pool) -> int:
    g = C.c_uint64()
    _lib.check(_lib.load().pkv_pool_generation(pool._h, C.addressof(g)), "pkv_pool_generation")
    return g.value



@on_device(lambda queries, store, *a, **k: store.device)
def paged_attention(queries, store: KvStore, meta: MaskMeta, config: AttentionConfig, *,
                    stats: KernelStats | None = None, block_mask: BlockMask | None = None,
                    skip_empty: bool = True, out_dtype=None, precision: str = "auto"):
    """Exact attention over scattered pages (attention.py:332-354), on the GPU.

    `queries` is (n_queries, head_count, head_dim), numpy or torch; the result
    is a device tensor (fp32 unless `out_dtype` says otherwise).
    `precision`: "auto" runs bf16 caches on the tensor-core kernel (P rounded
    to bf16; 2e-2 contract) and fp32/fp16 caches on the fp32 CUDA-core kernel
    (1e-5 contract); "exact" forces the CUDA-core kernel, "tensor" the
    tensor-core ones, "prefill" the K3 tcgen05 prefill kernel.  Suffix /
    self-attention metas over bf16 caches (fp16 under "tensor") with query
    runs of >= PREFILL_MIN_RUN positions go to K3."""
    import torch

    if stats is None and block_mask is None:
        out = _prefill_fast(queries, store, meta, config, out_dtype, precision)
        if out is not None:
            return out
    _check_queries(queries, meta, config)
    if store.head_count != config.kv_head_count or store.head_dim != config.head_dim:
        raise ShapeMismatch("store head layout does not match attention config")
    if config.page_size != store.page_size:
        raise ShapeMismatch("attention page_size does not match the pool")
    view = meta.view
    gen = _pool_generation(store.pool)  # read before the tables: a later change invalidates the memo
    n_pages, seq_row = store.pool.tables_info(view.ids)  # one native call for every table
    lengths = np.asarray(view.lengths, dtype=np.int64)
    bad = np.nonzero((lengths < 0) | (lengths > n_pages * store.page_size))[0]
    if bad.size:
        i = int(bad[0])
        raise OutOfRange(f"length {int(lengths[i])} exceeds reserved capacity of sequence {view.ids[i]!r}")
    # a suffix-shaped meta (the K3 route) always has >= 1 allowed key per query
    route = _prefill_route(meta, config, store.dtype_code, precision, seq_row)
    nkeys = None
    if route is None or stats is not None:
        nkeys = allowed_key_counts(meta, config.causal)
        if meta.query_count and (nkeys <= 0).any():
            bad = np.nonzero(nkeys <= 0)[0].tolist()
            raise NoAllowedKeys(f"queries {bad} have zero allowed keys")
        if stats is not None:
            _fill_stats(stats, meta, config, nkeys, block_mask)
    device = store.device
    q, qcode = _q_tensor(queries, device)
    mirror = store.pool.device_table(device)
    if route is not None:
        rec = {} if stats is None and block_mask is None else None
        out = _launch_prefill(q, meta, config, None, k=store.k_cache, v=store.v_cache,
                              kv_code=store.dtype_code, bt=mirror, rows=seq_row,
                              out_dtype=out_dtype or torch.float32, device=device, route=route, memo=rec)
        if rec:
            _remember_prefill(queries, store, meta, config, out_dtype, precision, gen, rec)
        return out
    return _launch_attention(q, qcode, meta, config, nkeys, k=store.k_cache, v=store.v_cache,
                             kv_code=store.dtype_code, bt=mirror, bt_stride=mirror.shape[1],
                             seq_row=seq_row, seq_start=None,
                             out_dtype=out_dtype or torch.float32, device=device,
                             precision=precision)


def gathered_attention(queries, keys, values, meta: MaskMeta, config: AttentionConfig, *,
                       stats: KernelStats | None = None, block_mask: BlockMask | None = None,
                       skip_empty: bool = True, out_dtype=None, device=None, precision="auto"):
    """Same kernel over contiguous K/V (attention.py:357-378); bitwise equal to
    the paged path on identical content (the split schedule depends only on
    logical lengths)."""
    import torch

    from .store import _device

    _check_queries(queries, meta, config)
    expected = (meta.view.total_slots, config.kv_head_count, config.head_dim)
    if tuple(keys.shape) != expected or tuple(values.shape) != expected:
        raise ShapeMismatch(f"expected K/V of shape {expected}, got {tuple(keys.shape)}/{tuple(values.shape)}")
    nkeys = allowed_key_counts(meta, config.causal)
    if meta.query_count and (nkeys <= 0).any():
        raise NoAllowedKeys("a query has zero allowed keys")
    if stats is not None:
        _fill_stats(stats, meta, config, nkeys, block_mask)
    if device is None:
        device = keys.device if isinstance(keys, torch.Tensor) and keys.is_cuda else _device(None)
    k = to_device(keys, device)
    v = to_device(values, device, k.dtype)
    _, kv_code = torch_dtype(k.dtype)
    q, qcode = _q_tensor(queries, device)
    seq_start = meta.view.prefix_sums.astype(np.int64)
    route = _prefill_route(meta, config, kv_code, precision, seq_start)
    if route is not None:
        return _launch_prefill(q, meta, config, None, k=k, v=v, kv_code=kv_code, bt=None,
                               rows=seq_start, out_dtype=out_dtype or torch.float32, device=device,
                               route=route)
    return _launch_attention(q, qcode, meta, config, nkeys, k=k, v=v, kv_code=kv_code, bt=None,
                             bt_stride=0, seq_row=None, seq_start=seq_start,
                             out_dtype=out_dtype or torch.float32, device=device,
                             precision=precision)


# ---------------------------------------------------------------------------
# Dense float64 diagnostics (reference attention.py:389-474).  Not the hot
# path: plain torch math on the device, for API parity with the reference's
# oracle / instrumented mode.  GQA is accepted (kv head h // G), an extension.
# ---------------------------------------------------------------------------

def reference_attention(queries, keys, values, lengths, *, causal: bool = True, scale=None, q_lengths=None,
                        device=None):
    """attention.py:389-447: two-pass masked softmax in float64 over
    contiguous per-sequence K/V; the trailing q_lengths[s] positions of each
    sequence are the queries.  Returns float64 rows (device tensor)."""
    import torch

    from .store import _device

    # a diagnostic, not the hot path: device="cpu" is allowed
    dev = torch.device(device) if device is not None else (
        queries.device if isinstance(queries, torch.Tensor) and queries.is_cuda else _device(None))
    q = torch.as_tensor(np.asarray(queries) if not isinstance(queries, torch.Tensor) else queries).to(dev, torch.float64)
    k = torch.as_tensor(np.asarray(keys) if not isinstance(keys, torch.Tensor) else keys).to(dev, torch.float64)
    v = torch.as_tensor(np.asarray(values) if not isinstance(values, torch.Tensor) else values).to(dev, torch.float64)
    if q.ndim != 3 or k.shape != v.shape or k.ndim != 3:
        raise ShapeMismatch("queries/keys/values must be (rows, heads, head_dim)")
    if k.shape[2] != q.shape[2] or q.shape[1] % k.shape[1]:
        raise ShapeMismatch("queries and keys disagree on head layout")
    lengths = np.asarray(lengths, dtype=np.int64)
    if lengths.sum() != k.shape[0]:
        raise ShapeMismatch("lengths do not add up to the KV row count")
    q_lengths = lengths.copy() if q_lengths is None else np.asarray(q_lengths, dtype=np.int64)
    if q_lengths.shape != lengths.shape or (q_lengths < 0).any() or (q_lengths > lengths).any():
        raise ShapeMismatch("q_lengths must give 0 <= q_len <= len per sequence")
    if q.shape[0] != q_lengths.sum():
        raise ShapeMismatch("query rows do not match q_lengths")
    g = q.shape[1] // k.shape[1]
    scale = 1.0 / math.sqrt(q.shape[2]) if scale is None else float(scale)
    out = torch.empty_like(q)
    ko = qo = 0
    for n, ql in zip(lengths.tolist(), q_lengths.tolist()):
        if ql:
            kk = k[ko:ko + n].repeat_interleave(g, dim=1)
            vv = v[ko:ko + n].repeat_interleave(g, dim=1)
            s = torch.einsum("qhd,khd->hqk", q[qo:qo + ql], kk) * scale
            if causal:
                pos = torch.arange(n - ql, n, device=dev)
                s = s.masked_fill(torch.arange(n, device=dev)[None, :] > pos[:, None], float("-inf"))
            p = torch.softmax(s, dim=-1)
            out[qo:qo + ql] = torch.einsum("hqk,khd->qhd", p, vv)
        ko += n
        qo += ql
    return out


def attention_weights(queries, store: KvStore, meta: MaskMeta, config: AttentionConfig):
    """attention.py:450-474: the (n_queries, heads, kv_slots) float64 softmax
    weights over the paged content of the view, exactly zero on disallowed
    keys; raises NoAllowedKeys for a query without allowed keys."""
    import torch

    _check_queries(queries, meta, config)
    keys, _ = KvStore.gather_view(store, meta.view)  # device tensors (also under the numpy facade)
    dev = keys.device
    q = torch.as_tensor(np.asarray(queries) if not isinstance(queries, torch.Tensor) else queries).to(dev, torch.float64)
    g = config.head_count // config.kv_head_count
    k = keys.to(torch.float64).repeat_interleave(g, dim=1)
    s = torch.einsum("qhd,khd->qhk", q, k) * config.scale
    nk = allowed_key_counts(meta, config.causal)
    lo = meta.view.prefix_sums[meta.q_seq]
    slots = torch.arange(meta.view.total_slots, device=dev)
    lo_t = torch.as_tensor(lo, device=dev)[:, None]
    hi_t = lo_t + torch.as_tensor(nk, device=dev)[:, None]
    allow = (slots[None, :] >= lo_t) & (slots[None, :] < hi_t)
    if meta.query_count and (~allow.any(dim=1)).any():
        raise NoAllowedKeys("a query row has zero allowed keys")
    s = s.masked_fill(~allow[:, None, :], float("-inf"))
    p = torch.softmax(s, dim=-1)
    return torch.where(allow[:, None, :], p, torch.zeros((), dtype=p.dtype, device=dev))
