"""PagePool — drop-in for the reference allocator (reference pool.py:88-349).

The allocator state lives in the native library (csrc/pool.cpp): a mutex-
protected free stack, bump cursor, refcounts and block tables that reproduce
the reference's `dump()` bit-for-bit.  This module maps the reference's
arbitrary hashable sequence ids onto int64 handles, forwards clear/copy
callbacks to every attached store (clear-on-grant, pool.py:122-126; page
copies, pool.py:112-120) and keeps the device block-table mirror current.
"""

from __future__ import annotations

import ctypes as C
import itertools
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import UnknownSequence

MAX_POOL_PAGES = 1 << 32  # reference pool.py:36 — 32-bit block-table entries


@dataclass(frozen=True)
class PageAddress:
    """Physical location of one token slot (pool.py:39-47)."""

    page_id: int
    offset: int

    def flat(self, page_size: int) -> int:
        return self.page_id * page_size + self.offset


@dataclass(frozen=True)
class PoolCensus:
    """live + free + never == capacity (pool.py:74-85)."""

    capacity_pages: int
    live_pages: int
    free_pages: int
    never_allocated: int

    @property
    def conserved(self) -> bool:
        return self.live_pages + self.free_pages + self.never_allocated == self.capacity_pages


class _Entries:
    """Live view of a table's uint32 entries (the reference's array('I'),
    pool.py:61): reads and writes go to the native table."""

    __slots__ = ("_t",)
    itemsize = 4
    typecode = "I"

    def __init__(self, table):
        self._t = table

    def _all(self) -> list:
        return self._t._pool._entries(self._t._handle)

    def __len__(self):
        return self._t._pool._table_len(self._t._handle)

    def __iter__(self):
        return iter(self._all())

    def __getitem__(self, idx):
        vals = self._all()
        return vals[idx]

    def __setitem__(self, idx, value):
        pool, h = self._t._pool, self._t._handle
        n = len(self)
        if isinstance(idx, slice):
            rng = range(*idx.indices(n))
            vals = [int(v) for v in value]
            if len(vals) != len(rng):
                raise ValueError("cannot resize a block table through slice assignment")
            for i, v in zip(rng, vals):
                pool._set_entry(h, i, v)
        else:
            pool._set_entry(h, int(idx), int(value))

    def __eq__(self, other):
        return self._all() == list(other)

    def tolist(self) -> list:
        return self._all()

    def __repr__(self):
        return f"array('I', {self._all()})"


class BlockTable:
    """Per-sequence ordered page ids + valid-token count (pool.py:50-71)."""

    __slots__ = ("seq_id", "_pool", "_handle")

    def __init__(self, pool: "PagePool", seq_id, handle: int):
        self.seq_id = seq_id
        self._pool = pool
        self._handle = handle

    @property
    def entries(self) -> _Entries:
        return _Entries(self)

    @entries.setter
    def entries(self, values):
        _Entries(self)[:] = values

    @property
    def logical_len(self) -> int:
        out = C.c_int64()
        _lib.call("pkv_pool_get_logical_len", self._pool._h, self._handle, C.byref(out))
        return out.value

    @logical_len.setter
    def logical_len(self, value: int) -> None:
        _lib.call("pkv_pool_set_logical_len", self._pool._h, self._handle, int(value))

    def capacity(self, page_size: int) -> int:
        return len(self.entries) * page_size

    @property
    def mirror_row(self) -> int:
        out = C.c_int32()
        _lib.call("pkv_pool_mirror_row", self._pool._h, self._handle, C.byref(out))
        return out.value

    def __repr__(self) -> str:
        return (f"BlockTable(seq_id={self.seq_id!r}, pages={list(self.entries)}, "
                f"logical_len={self.logical_len})")


class PagePool:
    """Drop-in PagePool(capacity_pages, page_size=64) (pool.py:88-110)."""

    def __init__(self, capacity_pages: int, page_size: int = 64):
        lib = _lib.load()
        if capacity_pages <= 0 or capacity_pages > MAX_POOL_PAGES:
            raise ValueError(f"capacity_pages must be in [1, 2^32], got {capacity_pages}")
        if page_size <= 0 or page_size & (page_size - 1):
            raise ValueError(f"page_size must be a positive power of two, got {page_size}")
        h = C.c_void_p()
        _lib.check(lib.pkv_pool_create(int(capacity_pages), int(page_size), C.byref(h)))
        self._h = h
        self.page_size = int(page_size)
        self.capacity_pages = int(capacity_pages)
        self._ids: dict = {}
        self._handles = itertools.count(1)
        self._stores: list = []
        self._mirror = None  # torch int32 [rows, cols] on the stores' device
        self._mq_pending, self._mq_full = C.c_int64(), C.c_int32()
        # drain -> apply-enqueue is one critical section: a thread that finds
        # nothing pending must not launch before another thread's apply of
        # the cells it drained
        self._mirror_lock = threading.RLock()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().pkv_pool_destroy(h)
            except Exception:
                pass
            self._h = C.c_void_p()

    # -- storage hookup -----------------------------------------------------
    def attach_store(self, store) -> None:
        self._stores.append(store)

    def _clear_pages(self, pages) -> None:
        if pages:
            for s in self._stores:
                s.clear_pages(pages)

    def _copy_rows(self, src: int, dst: int, rows: int) -> None:
        for s in self._stores:
            s.copy_rows(src, dst, rows)

    def _copy_pages(self, triples) -> None:
        """Batched page copies (one K0b launch per attached store)."""
        for s in self._stores:
            s.copy_pages(triples)

    # -- handle mapping -------------------------------------------------------
    def _handle_or_ghost(self, seq_id) -> int:
        h = self._ids.get(seq_id)
        return -1 if h is None else h  # -1 never exists natively -> UnknownSequence

    def _entries(self, h: int) -> list:
        n = self._table_len(h)
        buf = (C.c_uint32 * max(n, 1))()
        _lib.call("pkv_pool_table_entries", self._h, h, buf, n)
        return list(buf[:n])

    def _table_len(self, h: int) -> int:
        out = C.c_int64()
        _lib.call("pkv_pool_table_len", self._h, h, C.byref(out))
        return out.value

    def _set_entry(self, h: int, idx: int, value: int) -> None:
        if not 0 <= value < (1 << 32):
            raise OverflowError("unsigned int is greater than maximum")
        _lib.call("pkv_pool_table_set_entry", self._h, h, idx, value)

    # -- sequence lifecycle -----------------------------------------------------
    def pages_for(self, length: int) -> int:
        return -(-length // self.page_size)

    def reserve(self, seq_id, length: int) -> list[int]:
        """pool.py:154-174; granted pages are zeroed in every attached store."""
        existing = seq_id in self._ids
        h = self._ids[seq_id] if existing else next(self._handles)
        # the native side never grants more than the pool holds: an oversized
        # request fails there with CapacityExhausted, not here with MemoryError
        n_max = max(min(self.pages_for(length), self.capacity_pages), 1) if length >= 0 else 1
        buf = (C.c_uint32 * n_max)()
        n = C.c_int64()
        _lib.call("pkv_pool_reserve", self._h, h, int(length), buf, C.byref(n))
        self._ids[seq_id] = h
        pages = list(buf[:n.value])
        self._clear_pages(pages)
        return pages

    def grow(self, seq_id, new_len: int) -> list[int]:
        """pool.py:176-187; no-op when capacity already covers new_len."""
        h = self._handle_or_ghost(seq_id)
        n_max = max(min(self.pages_for(new_len), self.capacity_pages), 1)
        buf = (C.c_uint32 * n_max)()
        n = C.c_int64()
        _lib.call("pkv_pool_grow", self._h, h, int(new_len), buf, C.byref(n))
        pages = list(buf[:n.value])
        self._clear_pages(pages)
        return pages

    def free(self, seq_id) -> int:
        """pool.py:189-199; returns the number of pages reclaimed."""
        h = self._handle_or_ghost(seq_id)
        n = C.c_int64()
        try:
            _lib.call("pkv_pool_free", self._h, h, C.byref(n))
        finally:
            if h != -1 and not self._has(h):
                self._ids.pop(seq_id, None)
        return n.value

    def fork(self, parent_seq, child_seq, prefix_len: int) -> BlockTable:
        """pool.py:201-236; a partial trailing page is copied in every store."""
        ph = self._handle_or_ghost(parent_seq)
        existing = child_seq in self._ids
        ch = self._ids[child_seq] if existing else next(self._handles)
        src, dst, rows = C.c_int64(), C.c_int64(), C.c_int64()
        try:
            _lib.call("pkv_pool_fork", self._h, ph, ch, int(prefix_len), C.byref(src),
                      C.byref(dst), C.byref(rows))
        finally:
            if not existing and self._has(ch):
                self._ids[child_seq] = ch  # registered even on a late IndexError
        if dst.value >= 0:
            self._copy_rows(src.value, dst.value, rows.value)
        return BlockTable(self, child_seq, ch)

    def privatize(self, seq_id, block_idx: int):
        """pool.py:238-254 copy-on-write; returns the fresh page or None."""
        h = self._handle_or_ghost(seq_id)
        old, new = C.c_int64(), C.c_int64()
        _lib.call("pkv_pool_privatize", self._h, h, int(block_idx), C.byref(old), C.byref(new))
        if new.value < 0:
            return None
        self._copy_rows(old.value, new.value, self.page_size)
        return new.value

    def privatize_blocks(self, seq_id, blocks: np.ndarray) -> int:
        """store.py:143-145: privatize `blocks` (ascending) in one native call;
        performs the page copies and returns how many there were."""
        h = self._handle_or_ghost(seq_id)
        blocks = np.ascontiguousarray(blocks, dtype=np.int64)
        copies = np.empty(2 * max(blocks.size, 1), dtype=np.int64)
        n = C.c_int64()
        st = _lib.load().pkv_pool_privatize_blocks(self._h, h, blocks.ctypes.data, blocks.size,
                                                     copies.ctypes.data, C.byref(n))
        if n.value:  # copies of the blocks privatized before any failure, one launch per store
            pairs = copies[: 2 * n.value].reshape(-1, 2)
            self._copy_pages(np.column_stack([pairs, np.full(n.value, self.page_size)]))
        _lib.check(st, "pkv_pool_privatize_blocks")
        return n.value

    # -- addressing --------------------------------------------------------------
    def translate(self, seq_id, position: int) -> PageAddress:
        h = self._handle_or_ghost(seq_id)
        page, off = C.c_uint32(), C.c_uint32()
        _lib.call("pkv_pool_translate", self._h, h, int(position), C.byref(page), C.byref(off))
        return PageAddress(page.value, off.value)

    # -- introspection -------------------------------------------------------------
    def _has(self, h: int) -> bool:
        out = C.c_int32()
        _lib.call("pkv_pool_has_sequence", self._h, h, C.byref(out))
        return bool(out.value)

    def table(self, seq_id) -> BlockTable:
        h = self._ids.get(seq_id)
        if h is None:
            raise UnknownSequence(f"no block table for sequence {seq_id!r}")
        return BlockTable(self, seq_id, h)

    def tables_info(self, seq_ids):
        """(pages held int64[n], mirror row int32[n]) of the given sequences in
        one native call (pkv_pool_tables_info) — the per-call table lookups
        of the attention entry points, batched."""
        n = len(seq_ids)
        try:
            handles = np.fromiter((self._ids[s] for s in seq_ids), dtype=np.int64, count=n)
        except KeyError as e:
            raise UnknownSequence(f"no block table for sequence {e.args[0]!r}") from None
        pages = np.empty(n, dtype=np.int64)
        rows = np.empty(n, dtype=np.int32)
        _lib.call("pkv_pool_tables_info", self._h, handles.ctypes.data, n, pages.ctypes.data, rows.ctypes.data)
        return pages, rows

    def has_sequence(self, seq_id) -> bool:
        return seq_id in self._ids

    def sequences(self) -> list:
        n = C.c_int64()
        _lib.call("pkv_pool_sequence_count", self._h, C.byref(n))
        buf = (C.c_int64 * max(n.value, 1))()
        _lib.call("pkv_pool_sequences", self._h, buf, n.value)
        by_handle = {h: s for s, h in self._ids.items()}
        return [by_handle[h] for h in buf[:n.value]]

    def page_refcount(self, page_id: int) -> int:
        out = C.c_int64()
        _lib.call("pkv_pool_refcount", self._h, int(page_id), C.byref(out))
        return out.value

    def _census5(self):
        out = (C.c_int64 * 5)()
        _lib.call("pkv_pool_census", self._h, out)
        return list(out)

    @property
    def bump_cursor(self) -> int:
        return self._census5()[4]

    @property
    def free_page_count(self) -> int:
        return self._census5()[2]

    @property
    def available_pages(self) -> int:
        c = self._census5()
        return c[2] + c[3]

    def census(self) -> PoolCensus:
        cap, live, free, never, _ = self._census5()
        return PoolCensus(capacity_pages=cap, live_pages=live, free_pages=free, never_allocated=never)

    def free_stack(self) -> list:
        n = C.c_int64()
        _lib.call("pkv_pool_free_stack", self._h, None, 0, C.byref(n))
        buf = (C.c_uint32 * max(n.value, 1))()
        _lib.call("pkv_pool_free_stack", self._h, buf, n.value, C.byref(n))
        return list(buf[:n.value])

    def dump(self) -> dict:
        """Deterministic snapshot, same structure as pool.py:309-329."""
        census = self.census()
        tables = {}
        for seq_id in sorted(self._ids, key=repr):
            t = self.table(seq_id)
            tables[repr(seq_id)] = {"entries": self._entries(t._handle), "logical_len": t.logical_len}
        return {
            "page_size": self.page_size,
            "capacity_pages": self.capacity_pages,
            "bump_cursor": self.bump_cursor,
            "free_stack": self.free_stack(),
            "census": {
                "live_pages": census.live_pages,
                "free_pages": census.free_pages,
                "never_allocated": census.never_allocated,
            },
            "tables": tables,
        }

    # -- device block-table mirror ------------------------------------------------
    def device_table(self, device):
        """Bring the device mirror up to date and return it (int32 [rows, cols]).

        Dirty cells are drained from the native pool and applied by one small
        kernel; a shape change re-uploads the whole matrix."""
        import torch

        with self._mirror_lock:
            if device.index is not None and torch.cuda.current_device() != device.index:
                with torch.cuda.device(device):
                    return self._device_table(device)
            return self._device_table(device)

    def _device_table(self, device):
        import torch

        lib = _lib.load()
        pending, full = self._mq_pending, self._mq_full
        _lib.check(lib.pkv_pool_mirror_pending(self._h, C.byref(pending), C.byref(full)))
        m = self._mirror
        if not pending.value and not full.value and m is not None and m.device == device:
            return m  # fast path: nothing changed since the last call
        rows, cols = C.c_int64(), C.c_int64()
        _lib.check(lib.pkv_pool_mirror_shape(self._h, C.byref(rows), C.byref(cols)))
        if full.value or m is None or tuple(m.shape) != (rows.value, cols.value) or m.device != device:
            host = np.empty((rows.value, cols.value), dtype=np.int32)
            _lib.check(lib.pkv_pool_mirror_export(
                self._h, host.ctypes.data_as(C.POINTER(C.c_int32)), rows.value, cols.value))
            self._mirror = torch.from_numpy(host).to(device)
            return self._mirror
        if pending.value:
            pairs = np.empty((pending.value, 2), dtype=np.int32)
            n = C.c_int64()
            _lib.check(lib.pkv_pool_mirror_drain(
                self._h, pairs.ctypes.data_as(C.POINTER(C.c_int32)), pending.value, C.byref(n),
                C.byref(full)))
            # pageable source: the copy is staged before returning, no stream sync
            dev_pairs = torch.from_numpy(pairs[:n.value]).to(device, non_blocking=True)
            stream = torch.cuda.current_stream(device).cuda_stream
            _lib.check(lib.pkv_mirror_apply(C.c_void_p(m.data_ptr()), C.c_void_p(dev_pairs.data_ptr()),
                                            n.value, C.c_void_p(stream)), "pkv_mirror_apply")
        return m

    def mirror_row(self, seq_id) -> int:
        return self.table(seq_id).mirror_row
