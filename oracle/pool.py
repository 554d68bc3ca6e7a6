"""Oracle restatement of the reference page allocator (TEST INFRASTRUCTURE).

Follows `pkg/src/pagedkv/pool.py` of the reference.  Every observable of the
reference's `PagePool.dump()` (pool.py:309-329) is reproduced bit-exactly,
including the quirks SURVEY.md Appendix A lists:

* A.1 a failed multi-page grant pushes the pages it had already taken back
  onto the free stack in *taken order* (pool.py:143-148), so a failure can
  reverse the stack and migrate bumped pages into it; the raw bump counter
  overshoots by one per failed bump and is clamped when observed
  (pool.py:130-136, 286-290);
* A.2 LIFO reuse (free pushes in table order, pool.py:339-349);
* A.3 clear-on-grant into every attached store (pool.py:122-126);
* A.4 fork takes its copy page before sharing (pool.py:216-235); privatize is
  a full-page copy (pool.py:238-254).
"""

from __future__ import annotations

from .errors import (
    CapacityExhausted,
    DuplicateSequence,
    InvalidPrefix,
    OutOfRange,
    UnknownSequence,
)

MAX_POOL_PAGES = 1 << 32  # pool.py:36


class _Table:
    """Block table: uint32 page ids in logical order + valid-token count
    (pool.py:50-71)."""

    __slots__ = ("seq_id", "entries", "logical_len")

    def __init__(self, seq_id):
        self.seq_id = seq_id
        self.entries: list[int] = []
        self.logical_len = 0


class OraclePool:
    """pool.py:88-349 restated with plain Python containers."""

    def __init__(self, capacity_pages: int, page_size: int = 64):
        # pool.py:97-102
        if not 1 <= capacity_pages <= MAX_POOL_PAGES:
            raise ValueError("capacity_pages out of range")
        if page_size <= 0 or (page_size & (page_size - 1)) != 0:
            raise ValueError("page_size must be a positive power of two")
        self.page_size = page_size
        self.capacity_pages = capacity_pages
        self.free_stack: list[int] = []  # right end is the top (deque.pop)
        self.bump_raw = 0  # itertools.count value, may overshoot capacity
        self.refs: dict[int, int] = {}  # page -> refcount (absent == 0)
        self.tables: dict[object, _Table] = {}
        self.stores: list = []

    # ---- grants (pool.py:130-150) --------------------------------------
    def _grant_one(self):
        if self.free_stack:
            return self.free_stack.pop()
        page = self.bump_raw
        self.bump_raw += 1  # consumed even when it fails (overshoot)
        return page if page < self.capacity_pages else None

    def _grant(self, count: int) -> list[int]:
        got: list[int] = []
        while len(got) < count:
            page = self._grant_one()
            if page is None:
                self.free_stack.extend(got)  # A.1: taken order, not reversed
                raise CapacityExhausted(f"need {count} pages")
            got.append(page)
        return got

    def _set_ref(self, pages, value):
        for p in pages:
            self.refs[p] = value

    def _notify_clear(self, pages):
        for s in self.stores:
            s.clear_pages(pages)

    def _notify_copy(self, src, dst, rows):
        for s in self.stores:
            s.copy_rows(src, dst, rows)

    def _release(self, pages) -> int:
        # pool.py:339-349 — table order, push on reaching zero
        n = 0
        for p in pages:
            p = int(p)
            left = self.refs.get(p, 0) - 1
            if left:
                self.refs[p] = left
            else:
                self.refs.pop(p, None)
                self.free_stack.append(p)
                n += 1
        return n

    def _lookup(self, seq_id) -> _Table:
        t = self.tables.get(seq_id)
        if t is None:
            raise UnknownSequence(repr(seq_id))
        return t

    # ---- public ops ----------------------------------------------------
    def pages_for(self, length: int) -> int:
        return -(-length // self.page_size)

    def reserve(self, seq_id, length: int) -> list[int]:  # pool.py:154-174
        if length < 0:
            raise ValueError("negative length")
        if seq_id in self.tables:
            raise DuplicateSequence(repr(seq_id))
        t = _Table(seq_id)
        self.tables[seq_id] = t
        try:
            pages = self._grant(self.pages_for(length))
        except CapacityExhausted:
            del self.tables[seq_id]
            raise
        self._set_ref(pages, 1)
        self._notify_clear(pages)
        t.entries.extend(pages)
        return pages

    def grow(self, seq_id, new_len: int) -> list[int]:  # pool.py:176-187
        t = self._lookup(seq_id)
        missing = self.pages_for(new_len) - len(t.entries)
        if missing <= 0:
            return []
        pages = self._grant(missing)
        self._set_ref(pages, 1)
        self._notify_clear(pages)
        t.entries.extend(pages)
        return pages

    def free(self, seq_id) -> int:  # pool.py:189-199
        t = self.tables.pop(seq_id, None)
        if t is None:
            raise UnknownSequence(repr(seq_id))
        return self._release(t.entries)

    def fork(self, parent_seq, child_seq, prefix_len: int) -> _Table:
        # pool.py:201-236; check order: parent, prefix<0, InvalidPrefix, dup
        parent = self._lookup(parent_seq)
        if prefix_len < 0:
            raise ValueError("negative prefix")
        if prefix_len > parent.logical_len:
            raise InvalidPrefix(f"{prefix_len} > {parent.logical_len}")
        if child_seq in self.tables:
            raise DuplicateSequence(repr(child_seq))
        child = _Table(child_seq)
        self.tables[child_seq] = child
        whole, tail = divmod(prefix_len, self.page_size)
        copy_page = None
        if tail:
            try:
                copy_page = self._grant(1)[0]
            except CapacityExhausted:
                del self.tables[child_seq]
                raise
        shared = list(parent.entries[:whole])
        for p in shared:
            self.refs[p] = self.refs.get(p, 0) + 1
        child.entries.extend(shared)
        if copy_page is not None:
            self.refs[copy_page] = 1
            self._notify_copy(parent.entries[whole], copy_page, tail)
            child.entries.append(copy_page)
        child.logical_len = prefix_len
        return child

    def privatize(self, seq_id, block_idx: int):  # pool.py:238-254
        t = self._lookup(seq_id)
        old = int(t.entries[block_idx])
        if self.refs.get(old, 0) <= 1:
            return None
        new = self._grant(1)[0]
        self.refs[new] = 1
        self._notify_copy(old, new, self.page_size)
        t.entries[block_idx] = new
        self._release([old])
        return new

    def translate(self, seq_id, position: int) -> tuple[int, int]:
        # pool.py:258-266 -> (page_id, offset)
        t = self._lookup(seq_id)
        blk, off = divmod(position, self.page_size)
        if position < 0 or blk >= len(t.entries):
            raise OutOfRange(f"position {position}")
        return int(t.entries[blk]), off

    def table(self, seq_id) -> _Table:
        return self._lookup(seq_id)

    @property
    def bump_cursor(self) -> int:
        return min(self.bump_raw, self.capacity_pages)

    def census(self) -> dict:
        return {
            "live_pages": len(self.refs),
            "free_pages": len(self.free_stack),
            "never_allocated": self.capacity_pages - self.bump_cursor,
        }

    def dump(self) -> dict:
        # pool.py:309-329 — identical key set and ordering rules
        return {
            "page_size": self.page_size,
            "capacity_pages": self.capacity_pages,
            "bump_cursor": self.bump_cursor,
            "free_stack": list(self.free_stack),
            "census": self.census(),
            "tables": {
                repr(k): {
                    "entries": [int(e) for e in self.tables[k].entries],
                    "logical_len": int(self.tables[k].logical_len),
                }
                for k in sorted(self.tables, key=repr)
            },
        }
