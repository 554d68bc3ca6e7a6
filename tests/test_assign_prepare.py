"""pkv_pool_assign_prepare: the native host pass of KvStore.assign
(store.py:117-150) -- position scan, capacity check and ascending
copy-on-write -- against the per-block privatize loop on a twin pool."""
import ctypes as C

import numpy as np
import pytest

from paper_2506_07311_b200 import PagePool, _lib


def _prepare(pool, seq, positions):
    pos = np.ascontiguousarray(positions, dtype=np.int64)
    info = np.empty(5, dtype=np.int64)
    copies = np.empty(2 * max(pos.size, 1) + 2, dtype=np.int64)
    n = C.c_int64()
    _lib.check(_lib.load().pkv_pool_assign_prepare(pool._h, pool.table(seq)._handle, pos.ctypes.data, pos.size,
                                                   info.ctypes.data, copies.ctypes.data, copies.size,
                                                   C.addressof(n)))
    return info.tolist(), copies[: 2 * n.value].reshape(-1, 2).tolist()


def _forked_pair(ps=4):
    pools = []
    for _ in range(2):
        p = PagePool(64, page_size=ps)
        p.reserve("a", 10 * ps)
        p.table("a").logical_len = 10 * ps
        p.fork("a", "b", 6 * ps)  # b shares a's first six pages
        p.grow("b", 10 * ps)
        pools.append(p)
    return pools


def test_flags_and_bounds():
    pool = PagePool(32, page_size=4)
    pool.reserve("s", 20)
    info, copies = _prepare(pool, "s", np.arange(3, 11))
    assert info[:3] == [3, 10, _lib.PKV_ASSIGN_INCREASING | _lib.PKV_ASSIGN_CONTIGUOUS]
    assert info[3] == 5 and info[4] == pool.table("s").mirror_row and copies == []
    info, _ = _prepare(pool, "s", [1, 5, 9])
    assert info[2] == _lib.PKV_ASSIGN_INCREASING
    info, _ = _prepare(pool, "s", [5, 1, 5])
    assert info[:3] == [1, 5, 0]
    info, _ = _prepare(pool, "s", [0, 20])
    assert info[2] & _lib.PKV_ASSIGN_OUT_OF_RANGE
    info, _ = _prepare(pool, "s", [-1, 2])
    assert info[2] & _lib.PKV_ASSIGN_OUT_OF_RANGE


@pytest.mark.parametrize("positions", [np.arange(0, 40), np.arange(5, 19), [2, 3, 9, 17, 22, 23], [21]])
def test_cow_matches_privatize_loop(positions):
    ps = 4
    native, twin = _forked_pair(ps)
    info, copies = _prepare(native, "b", positions)
    blocks = np.unique(np.asarray(positions) // ps)
    expect = []
    for b in blocks:
        old = twin.table("b").entries[b]
        fresh = twin.privatize("b", int(b))
        if fresh is not None:
            expect.append([old, fresh])
    assert copies == expect
    assert native.dump() == twin.dump()


def test_out_of_range_and_unsorted_privatize_nothing():
    native, _ = _forked_pair()
    before = native.dump()
    info, copies = _prepare(native, "b", [0, 400])
    assert info[2] & _lib.PKV_ASSIGN_OUT_OF_RANGE and copies == [] and native.dump() == before
    info, copies = _prepare(native, "b", [3, 1])
    assert info[2] == 0 and copies == [] and native.dump() == before
