"""ctypes binding of libpkv200.so (the C ABI of include/pkv200.h).

This is the reference-side binding a Python caller adds: it
loads the in-tree library, declares every entry point and turns non-zero
status codes into the reference's exception classes.  There is no fallback —
a missing library raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# PKV200_LIB overrides the library (kernel-variant experiments); default in-tree
LIB_PATH = os.environ.get("PKV200_LIB") or os.path.join(_HERE, "libpkv200.so")

PKV_F32, PKV_F16, PKV_BF16 = 0, 1, 2
PKV_ASSIGN_INCREASING, PKV_ASSIGN_CONTIGUOUS, PKV_ASSIGN_OUT_OF_RANGE = 1, 2, 4
PREFILL_ITEM_INTS = 10  # {q_row0, cnt_a, cnt_b, qpos0, kv_len, row, kv_head, tiles_a, tiles_b, 0}

_STATUS = {
    1: errors.CapacityExhausted,
    2: errors.DuplicateSequence,
    3: errors.UnknownSequence,
    4: errors.InvalidPrefix,
    5: errors.OutOfRange,
    6: errors.ShapeMismatch,
    7: errors.NoAllowedKeys,
    8: ValueError,
    9: IndexError,
    10: errors.ConfigError,
    11: errors.DeviceError,
}

_i32, _i64, _u32, _u64, _f32, _vp = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float, C.c_void_p
_P = C.POINTER


class AttentionArgs(C.Structure):
    _fields_ = [
        ("q", _vp), ("q_dtype", _i32), ("n_queries", _i64),
        ("q_seq", _vp), ("q_nkeys", _vp),
        ("k_cache", _vp), ("v_cache", _vp), ("kv_dtype", _i32),
        ("block_table", _vp), ("bt_stride", _i64), ("seq_row", _vp), ("seq_start", _vp),
        ("page_size", _i32), ("hq", _i32), ("hkv", _i32), ("head_dim", _i32),
        ("scale", _f32), ("out", _vp), ("out_dtype", _i32),
        ("workspace", _vp), ("workspace_bytes", _i64),
        ("num_sms", _i32), ("target_waves", _i32),
        ("prof_start", _vp), ("prof_stop", _vp),
        ("mode", _i32), ("k_new", _vp), ("v_new", _vp),
        ("plan", _vp), ("plan_host", _vp),
        ("meta_host", _vp), ("meta_dev", _vp), ("meta_bytes", _i64),
    ]


class PrefillArgs(C.Structure):
    _fields_ = [
        ("q", _vp), ("total_q", _i64), ("k_cache", _vp), ("v_cache", _vp), ("kv_dtype", _i32),
        ("cache_rows", _i64), ("block_table", _vp), ("bt_stride", _i64), ("page_size", _i32),
        ("hq", _i32), ("hkv", _i32), ("head_dim", _i32), ("scale", _f32), ("causal", _i32),
        ("out", _vp), ("out_dtype", _i32), ("plan", _vp), ("n_items", _i64),
        ("prof_start", _vp), ("prof_stop", _vp), ("debug", _vp),
    ]


class StepStageArgs(C.Structure):
    _fields_ = [
        ("pool", _vp), ("seqs", _vp), ("n", _i64), ("page_size", _i32), ("hq", _i32), ("hkv", _i32),
        ("meta_host", _vp), ("meta_dev", _vp), ("meta_cap", _i64), ("slot_event", _vp),
        ("n_stores", _i32), ("k_caches", _vp), ("v_caches", _vp), ("row_bytes", _i64),
        ("mirror_dev", _vp), ("mirror_rows", _i64), ("mirror_cols", _i64),
        ("meta_used", _i64), ("needs_resync", _i32), ("launches", _i32),
        ("n_granted", _i64), ("granted_off", _i64), ("n_copies", _i64), ("copies_off", _i64),
    ]


class DecodeIO(C.Structure):
    _fields_ = [
        ("q_host", _vp), ("k_host", _vp), ("v_host", _vp), ("out_host", _vp),
        ("q_bytes", _i64), ("kv_bytes", _i64), ("out_bytes", _i64), ("launched", _i32), ("launches", _i32),
    ]


# name -> (restype, argtypes); every symbol the header declares
SIGNATURES = {
    "pkv_last_error": (C.c_char_p, []),
    "pkv_abi_version": (C.c_int, []),
    "pkv_pool_create": (C.c_int, [_u64, _u32, _P(_vp)]),
    "pkv_pool_destroy": (None, [_vp]),
    "pkv_pool_reserve": (C.c_int, [_vp, _i64, _i64, _P(_u32), _P(_i64)]),
    "pkv_pool_grow": (C.c_int, [_vp, _i64, _i64, _P(_u32), _P(_i64)]),
    "pkv_pool_free": (C.c_int, [_vp, _i64, _P(_i64)]),
    "pkv_pool_fork": (C.c_int, [_vp, _i64, _i64, _i64, _P(_i64), _P(_i64), _P(_i64)]),
    "pkv_pool_privatize": (C.c_int, [_vp, _i64, _i64, _P(_i64), _P(_i64)]),
    "pkv_pool_privatize_blocks": (C.c_int, [_vp, _i64, _vp, _i64, _vp, _P(_i64)]),
    "pkv_pool_prepare_append": (C.c_int, [_vp, _P(_i64), _i64, _P(_i32), _P(_i32), _P(_u32), _i64,
                                          _P(_i64), _P(_i64)]),
    "pkv_pool_translate": (C.c_int, [_vp, _i64, _i64, _P(_u32), _P(_u32)]),
    "pkv_pool_has_sequence": (C.c_int, [_vp, _i64, _P(_i32)]),
    "pkv_pool_table_len": (C.c_int, [_vp, _i64, _P(_i64)]),
    "pkv_pool_table_entries": (C.c_int, [_vp, _i64, _P(_u32), _i64]),
    "pkv_pool_table_set_entry": (C.c_int, [_vp, _i64, _i64, _u32]),
    "pkv_pool_get_logical_len": (C.c_int, [_vp, _i64, _P(_i64)]),
    "pkv_pool_set_logical_len": (C.c_int, [_vp, _i64, _i64]),
    "pkv_pool_sequence_count": (C.c_int, [_vp, _P(_i64)]),
    "pkv_pool_sequences": (C.c_int, [_vp, _P(_i64), _i64]),
    "pkv_pool_refcount": (C.c_int, [_vp, _u64, _P(_i64)]),
    "pkv_pool_census": (C.c_int, [_vp, _P(_i64)]),
    "pkv_pool_free_stack": (C.c_int, [_vp, _P(_u32), _i64, _P(_i64)]),
    "pkv_pool_tables_info": (C.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "pkv_pool_generation": (C.c_int, [_vp, _vp]),
    "pkv_kv_assign": (C.c_int, [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp,
                                _i64, _vp, _vp]),
    "pkv_pool_assign_prepare": (C.c_int, [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp]),
    "pkv_prefill_plan_meta": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _i64,
                                        _vp, _vp, _vp]),
    "pkv_pool_mirror_row": (C.c_int, [_vp, _i64, _P(_i32)]),
    "pkv_pool_mirror_shape": (C.c_int, [_vp, _P(_i64), _P(_i64)]),
    "pkv_pool_mirror_drain": (C.c_int, [_vp, _P(_i32), _i64, _P(_i64), _P(_i32)]),
    "pkv_pool_mirror_pending": (C.c_int, [_vp, _P(_i64), _P(_i32)]),
    "pkv_pool_mirror_export": (C.c_int, [_vp, _P(_i32), _i64, _i64]),
    "pkv_mirror_apply": (C.c_int, [_vp, _vp, _i64, _vp]),
    "pkv_page_zero": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp]),
    "pkv_copy_h2d_record": (C.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "pkv_event_wait": (C.c_int, [_vp]),
    "pkv_page_copy1": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i32, _vp]),
    "pkv_page_copy": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i32, _vp]),
    "pkv_kv_append_range": (C.c_int, [_vp, _vp, _i64, _i32, _i32, _vp, _i64, _i32, _vp, _vp, _i64, _vp]),
    "pkv_kv_append": (C.c_int, [_vp, _vp, _i64, _vp, _i32, _vp, _vp, _i64, _i32, _vp, _vp, _i64, _vp]),
    "pkv_kv_gather": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _i64, _i64, _i32, _i64, _vp, _vp, _vp]),
    "pkv_attention_workspace_bytes": (_i64, [_i64, _i32, _i32]),
    "pkv_decode_step_stage_ints": (_i64, [_i64, _i32]),
    "pkv_decode_step_stage": (C.c_int, [_P(StepStageArgs), _vp]),
    "pkv_decode_step_prepare": (C.c_int, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _i64, _P(_i64), _vp, _i64,
                                          _P(_i64), _vp]),
    "pkv_attention_plan_ints": (_i64, [_i64, _i32]),
    "pkv_plan_memo_reset": (None, []),
    "pkv_attention_plan": (C.c_int, [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _i64, _P(_i64)]),
    "pkv_attention_plan_d": (C.c_int, [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _i64, _P(_i64)]),
    "pkv_paged_attention": (C.c_int, [_P(AttentionArgs), _vp]),
    "pkv_step_graph_create": (C.c_int, [_P(_vp)]),
    "pkv_step_graph_destroy": (None, [_vp]),
    "pkv_step_graph_stats": (C.c_int, [_vp, _P(_i64), _P(_i64)]),
    "pkv_decode_step_graph": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pkv_decode_step": (C.c_int, [_P(StepStageArgs), _P(AttentionArgs), _P(DecodeIO), _vp]),
    "pkv_prefill_supported": (C.c_int, [_i32, _i32, _i32, _i32, _i32]),
    "pkv_prefill_plan_ints": (_i64, [_vp, _i64, _i32, _i32]),
    "pkv_prefill_plan": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _i64, _P(_i64)]),
    "pkv_paged_prefill": (C.c_int, [_P(PrefillArgs), _vp]),
    "pkv_device_sm_count": (C.c_int, [_P(_i32)]),
    "pkv_debug_trace": (C.c_int, [_i32, _P(_u64), _i64]),
    "pkv_debug_inject_failure": (C.c_int, [_i32]),
    "pkv_debug_step_times": (C.c_int, [_P(_i64), _i32]),
}

PKV_FAIL_STEP_UPLOAD, PKV_FAIL_STEP_LAUNCH = 1, 2

_lib = None


def load() -> C.CDLL:
    """Load libpkv200.so once; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise errors.DeviceError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2506_07311_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = load().pkv_last_error().decode(errors="replace")
    exc = _STATUS.get(status, errors.DeviceError)
    raise exc(f"{what}: {msg}" if what and exc is errors.DeviceError else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def attention_plan(q_nkeys, q_row, page_size: int, hq: int, hkv: int, target_waves: int = 0,
                   head_dim: int = 128):
    """Host plan of the tensor-core decode (pkv_attention_plan_d) as int32 numpy."""
    import numpy as np

    nk = np.ascontiguousarray(q_nkeys, dtype=np.int32)
    rows = np.ascontiguousarray(q_row, dtype=np.int32)
    n = nk.size
    lib = load()
    out = np.empty(lib.pkv_attention_plan_ints(n, hq), dtype=np.int32)
    got = C.c_int64()
    check(lib.pkv_attention_plan_d(nk.ctypes.data, rows.ctypes.data, n, page_size, hq, hkv, head_dim, 0,
                                   target_waves, out.ctypes.data, out.size, C.byref(got)),
          "pkv_attention_plan_d")
    return out[: got.value].copy()


def prefill_plan(q_start, q_len, seq_len, seq_row, hq: int, hkv: int, causal: bool):
    """Host work plan of the tcgen05 prefill (pkv_prefill_plan) as int32 numpy
    [n_items, PREFILL_ITEM_INTS]."""
    import numpy as np

    qs = np.ascontiguousarray(q_start, dtype=np.int64)
    ql = np.ascontiguousarray(q_len, dtype=np.int32)
    sl = np.ascontiguousarray(seq_len, dtype=np.int32)
    sr = np.ascontiguousarray(seq_row, dtype=np.int32)
    lib = load()
    cap = int(lib.pkv_prefill_plan_ints(ql.ctypes.data, ql.size, hq, hkv))
    out = np.empty(max(cap, PREFILL_ITEM_INTS), dtype=np.int32)
    got = C.c_int64()
    check(lib.pkv_prefill_plan(qs.ctypes.data, ql.ctypes.data, sl.ctypes.data, sr.ctypes.data, ql.size,
                               hq, hkv, int(bool(causal)), out.ctypes.data, out.size, C.byref(got)),
          "pkv_prefill_plan")
    return out[: PREFILL_ITEM_INTS * got.value].reshape(-1, PREFILL_ITEM_INTS).copy()
