"""All-or-nothing decode-step staging (CPU).

The batched decode step (pkv_decode_step_stage) advances the allocator —
grow, copy-on-write, logical_len += 1 — and then uploads metadata and
launches.  A failure after the allocator moved must put it back exactly, the
reference's atomic-failure contract (pool.py:143-148, 165-169): dump(), the
free-stack order, refcounts and the device-mirror export all unchanged.

The failure is injected before any CUDA call (pkv_debug_inject_failure), so
this runs without a GPU; the GPU twin (tests/test_gpu_decode_tc.py) checks the
same through DecodeBatch.step.
"""

import ctypes as C

import numpy as np
import pytest

from paper_2506_07311_b200 import DeviceError, PagePool, _lib


def _mirror(pool):
    lib = _lib.load()
    rows, cols = C.c_int64(), C.c_int64()
    _lib.check(lib.pkv_pool_mirror_shape(pool._h, C.byref(rows), C.byref(cols)))
    out = np.zeros((rows.value, cols.value), dtype=np.int32)
    _lib.check(lib.pkv_pool_mirror_export(pool._h, out.ctypes.data_as(C.POINTER(C.c_int32)), rows.value,
                                          cols.value))
    return out


def _live_mirror(pool):
    """The mirror cells the kernels read: each live table's row up to its
    entry count (cells past it are don't-care)."""
    m = _mirror(pool)
    return {repr(s): m[pool.table(s).mirror_row, : len(pool.table(s).entries)].tolist()
            for s in pool.sequences()}


def _refcounts(pool):
    return [pool.page_refcount(p) for p in range(pool.capacity_pages)]


def _stage(pool, seq_ids, hq=8, hkv=2):
    lib = _lib.load()
    n = len(seq_ids)
    handles = np.asarray([pool.table(s)._handle for s in seq_ids], dtype=np.int64)
    width = int(lib.pkv_decode_step_stage_ints(n, hq))
    host = np.zeros(width, dtype=np.int32)
    a = _lib.StepStageArgs()
    a.pool, a.seqs, a.n = pool._h, handles.ctypes.data, n
    a.page_size, a.hq, a.hkv = pool.page_size, hq, hkv
    a.meta_host, a.meta_dev, a.meta_cap = host.ctypes.data, host.ctypes.data, width
    a.slot_event = None
    a.n_stores = 0
    a.mirror_dev = None
    return lib.pkv_decode_step_stage(C.byref(a), None), a, (handles, host)


def _scenario(seed):
    """A pool whose next decode step grows some tables (page boundary),
    copy-on-writes shared blocks (forks) and plain-appends the rest, with a
    scrambled free stack."""
    rng = np.random.default_rng(seed)
    pool = PagePool(96, page_size=4)
    lens = [int(x) for x in rng.integers(1, 30, 6)]
    lens[0] = 8  # next token opens a new page
    lens[2] = max(lens[2], 9)
    for i, n in enumerate(lens):
        pool.reserve(f"s{i}", n)
        pool.table(f"s{i}").logical_len = n
    for i in (1, 3):  # freed tables scramble the free stack
        pool.free(f"s{i}")
    pool.fork("s2", "c2", 8)  # two shared pages; the child's next write lands in one of them
    pool.table("c2").logical_len = 6
    pool.fork("s4", "c4", 4 * (pool.table("s4").logical_len // 4))  # page-aligned: child grows
    pool.table("c4").logical_len = 4 * (pool.table("s4").logical_len // 4)
    return pool, ["s0", "s2", "c2", "s4", "c4", "s5"]


@pytest.mark.parametrize("seed", range(4))
def test_injected_upload_failure_rolls_the_allocator_back(seed):
    pool, ids = _scenario(seed)
    before = (pool.dump(), _refcounts(pool), _live_mirror(pool))
    _lib.load().pkv_debug_inject_failure(_lib.PKV_FAIL_STEP_UPLOAD)
    st, _, _ = _stage(pool, ids)
    assert st != 0
    with pytest.raises(DeviceError, match="injected"):
        _lib.check(st, "pkv_decode_step_stage")
    after = (pool.dump(), _refcounts(pool), _live_mirror(pool))
    assert after == before
    for s, cells in after[2].items():  # the mirror agrees with the tables
        assert cells == before[0]["tables"][s]["entries"]
    assert pool.census().conserved


def _prepare_append(pool, seq_ids):
    """pkv_pool_prepare_append (host only): the allocator half of a step."""
    lib = _lib.load()
    n = len(seq_ids)
    handles = np.asarray([pool.table(s)._handle for s in seq_ids], dtype=np.int64)
    pos, rows = np.zeros(n, np.int32), np.zeros(n, np.int32)
    pages, copies = np.zeros(2 * n + 1, np.uint32), np.zeros(2 * n, np.int64)
    n_pages = C.c_int64()
    P = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    _lib.check(lib.pkv_pool_prepare_append(pool._h, P(handles, C.c_int64), n, P(pos, C.c_int32),
                                           P(rows, C.c_int32), P(pages, C.c_uint32), pages.size,
                                           C.byref(n_pages), P(copies, C.c_int64)))
    return pos.tolist(), pages[: n_pages.value].tolist(), copies.tolist()


@pytest.mark.parametrize("seed", range(4))
def test_step_after_rollback_equals_step_without_failure(seed):
    """The rolled-back pool then takes the step exactly as an untouched twin
    (same granted pages, copies, positions, dump and mirror)."""
    pool_a, ids = _scenario(seed)
    pool_b, _ = _scenario(seed)
    _lib.load().pkv_debug_inject_failure(_lib.PKV_FAIL_STEP_UPLOAD)
    assert _stage(pool_a, ids)[0] != 0
    got_a = _prepare_append(pool_a, ids)
    got_b = _prepare_append(pool_b, ids)
    assert got_a == got_b
    assert got_a[1] and any(c >= 0 for c in got_a[2])  # the scenario grows and copies
    assert pool_a.dump() == pool_b.dump()
    assert _live_mirror(pool_a) == _live_mirror(pool_b)
    assert _refcounts(pool_a) == _refcounts(pool_b)


def test_injection_is_one_shot_and_disarmable():
    lib = _lib.load()
    pool, ids = _scenario(0)

    def msg():
        return lib.pkv_last_error().decode()

    lib.pkv_debug_inject_failure(_lib.PKV_FAIL_STEP_UPLOAD)
    lib.pkv_debug_inject_failure(0)
    _stage(pool, ids)
    assert "injected" not in msg()
    pool, ids = _scenario(0)
    lib.pkv_debug_inject_failure(_lib.PKV_FAIL_STEP_UPLOAD)
    assert _stage(pool, ids)[0] != 0 and "injected" in msg()
    _stage(pool, ids)
    assert "injected" not in msg()


def test_capacity_failure_mutates_nothing():
    pool = PagePool(4, page_size=4)
    for i in range(4):
        pool.reserve(i, 4)
        pool.table(i).logical_len = 4
    before = pool.dump()
    st, _, _ = _stage(pool, [0, 1])
    assert st == 1  # CapacityExhausted
    assert pool.dump() == before
