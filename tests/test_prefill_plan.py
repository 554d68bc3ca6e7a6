"""Host side of K3 (no GPU): suffix-run detection and the work planner.

The planner cuts each sequence's query run (MaskMeta.self_attention /
.suffix, reference attention.py:81-110) into items of one kv head x 128/G
positions whose key range is the causal prefix of the item's last query.
"""

import numpy as np
import pytest

from paper_2506_07311_b200 import MaskMeta, OutOfRange
from paper_2506_07311_b200 import _lib
from paper_2506_07311_b200.attention import suffix_runs
from paper_2506_07311_b200.store import BatchView


def test_suffix_runs_accepts_self_attention_and_suffix():
    view = BatchView.from_lengths([5, 0, 3], ids=["a", "b", "c"])
    qs, ql = suffix_runs(MaskMeta.self_attention(view))
    assert qs.tolist() == [0, 5, 5] and ql.tolist() == [5, 0, 3]
    qs, ql = suffix_runs(MaskMeta.suffix(view, [2, 0, 3]))
    assert qs.tolist() == [0, 2, 2] and ql.tolist() == [2, 0, 3]


def test_suffix_runs_rejects_other_metas():
    view = BatchView.from_lengths([5, 3])
    assert suffix_runs(MaskMeta(view, q_seq=[0, 0], q_pos=[1, 2])) is None  # not ending at len-1
    assert suffix_runs(MaskMeta(view, q_seq=[0, 0], q_pos=[4, 4])) is None  # repeated position
    assert suffix_runs(MaskMeta.decode(view)) is not None  # decode is a run of one


def test_plan_items_cover_every_query_once():
    lens = np.array([1, 300, 129, 8192], dtype=np.int32)
    ql = np.array([1, 300, 100, 8192], dtype=np.int32)
    qs = np.concatenate([[0], np.cumsum(ql)[:-1]]).astype(np.int64)
    rows = np.array([3, 0, 7, 1], dtype=np.int32)
    hq, hkv = 32, 8
    plan = _lib.prefill_plan(qs, ql, lens, rows, hq, hkv, causal=True)
    qt = 128 // (hq // hkv)
    cover = np.zeros((int(ql.sum()), hkv), dtype=np.int64)
    for q_row0, cnt, pos0, kv_len, row, kvh, tiles, _ in plan:
        assert 1 <= cnt <= qt
        cover[q_row0:q_row0 + cnt, kvh] += 1
        s = int(np.searchsorted(qs, q_row0, side="right") - 1)
        assert kv_len == lens[s] and row == rows[s]
        assert pos0 == lens[s] - ql[s] + (q_row0 - qs[s])
        assert tiles == -(-min(pos0 + cnt, kv_len) // 128)
    assert (cover == 1).all()
    assert (np.diff(plan[:, 6]) <= 0).all()  # longest first


def test_plan_non_causal_visits_all_keys_and_validates():
    plan = _lib.prefill_plan([0], [10], [1000], [0], 8, 8, causal=False)
    assert plan.shape == (8, 8) and (plan[:, 6] == 8).all() and sorted(plan[:, 5]) == list(range(8))
    with pytest.raises(OutOfRange):
        _lib.prefill_plan([0], [20], [10], [0], 8, 8, causal=True)


def test_supported_shapes():
    lib = _lib.load()
    assert lib.pkv_prefill_supported(32, 8, 128, 16, _lib.PKV_BF16)
    assert lib.pkv_prefill_supported(8, 8, 64, 8, _lib.PKV_F16)
    assert not lib.pkv_prefill_supported(48, 2, 128, 16, _lib.PKV_BF16)  # G=24 does not divide 128
    assert not lib.pkv_prefill_supported(8, 8, 96, 16, _lib.PKV_BF16)
    assert not lib.pkv_prefill_supported(8, 8, 128, 4, _lib.PKV_BF16)
    assert not lib.pkv_prefill_supported(8, 8, 128, 16, _lib.PKV_F32)
