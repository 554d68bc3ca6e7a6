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
    assert plan.shape[1] == _lib.PREFILL_ITEM_INTS
    qt = 128 // (hq // hkv)
    cover = np.zeros((int(ql.sum()), hkv), dtype=np.int64)
    for q_row0, cnt_a, cnt_b, pos0, kv_len, row, kvh, tiles_a, tiles_b, _ in plan:
        assert 1 <= cnt_a <= qt and 0 <= cnt_b <= qt and (cnt_b == 0 or cnt_a == qt)
        s = int(np.searchsorted(qs, q_row0, side="right") - 1)
        assert kv_len == lens[s] and row == rows[s]
        assert pos0 == lens[s] - ql[s] + (q_row0 - qs[s])
        for t, (cnt, tiles) in enumerate(((cnt_a, tiles_a), (cnt_b, tiles_b))):
            cover[q_row0 + t * qt:q_row0 + t * qt + cnt, kvh] += 1
            want = -(-min(pos0 + t * qt + cnt, kv_len) // 128) if cnt else 0
            assert tiles == want
    assert (cover == 1).all()
    longest = np.maximum(plan[:, 7], plan[:, 8])
    assert (np.diff(longest) <= 0).all()  # longest first


def test_plan_non_causal_visits_all_keys_and_validates():
    plan = _lib.prefill_plan([0], [10], [1000], [0], 8, 8, causal=False)
    assert plan.shape == (8, _lib.PREFILL_ITEM_INTS) and (plan[:, 7] == 8).all() and (plan[:, 8] == 0).all()
    assert sorted(plan[:, 6]) == list(range(8))
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


@pytest.mark.timeout(300, method="thread")
def test_prefill_plan_fuzz_covers_every_query_once():
    """Random suffix metas (GQA groups 1-16, causal or not): every (query,
    kv head) lands in exactly one item half, tile counts follow the mask."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        hkv = int(rng.choice([1, 2, 4, 8]))
        g = int(rng.choice([1, 2, 4, 8, 16]))
        causal = bool(rng.integers(2))
        n = int(rng.integers(1, 9))
        lens = np.maximum(1, np.exp(rng.uniform(0, np.log(6000), n))).astype(np.int32)
        ql = np.asarray([int(rng.integers(1, x + 1)) for x in lens], dtype=np.int32)
        qs = np.concatenate([[0], np.cumsum(ql)[:-1]]).astype(np.int64)
        rows = rng.permutation(n).astype(np.int32)
        plan = _lib.prefill_plan(qs, ql, lens, rows, hkv * g, hkv, causal=causal)
        qt = 128 // g
        cover = np.zeros((int(ql.sum()), hkv), dtype=np.int64)
        for q_row0, cnt_a, cnt_b, pos0, kv_len, row, kvh, tiles_a, tiles_b, _ in plan:
            s = int(np.searchsorted(qs, q_row0, side="right") - 1)
            assert kv_len == lens[s] and row == rows[s]
            for t, (cnt, tiles) in enumerate(((cnt_a, tiles_a), (cnt_b, tiles_b))):
                cover[q_row0 + t * qt:q_row0 + t * qt + cnt, kvh] += 1
                if cnt:
                    keys = min(pos0 + t * qt + cnt, kv_len) if causal else kv_len
                    assert tiles == -(-keys // 128)
        assert (cover == 1).all()


def _metas():
    view = BatchView.from_lengths([5, 0, 3, 40], ids=["a", "b", "c", "d"])
    yield MaskMeta.self_attention(view)
    yield MaskMeta.suffix(view, [2, 0, 3, 17])
    yield MaskMeta.decode(BatchView.from_lengths([4, 9]))
    yield MaskMeta(BatchView.from_lengths([5, 3]), q_seq=[0, 0], q_pos=[1, 2])  # not ending at len-1
    yield MaskMeta(BatchView.from_lengths([5, 3]), q_seq=[0, 0], q_pos=[4, 4])  # repeated position
    yield MaskMeta(BatchView.from_lengths([5, 3]), q_seq=np.zeros(0, np.int64), q_pos=np.zeros(0, np.int64))


@pytest.mark.parametrize("causal", [True, False])
def test_native_route_matches_suffix_runs_and_planner(causal):
    """pkv_prefill_plan_meta (the one-pass K3 route) == suffix_runs + the planner."""
    from paper_2506_07311_b200 import AttentionConfig
    from paper_2506_07311_b200.attention import _prefill_plan_meta

    cfg = AttentionConfig(head_count=8, head_dim=64, page_size=16, kv_head_count=2, causal=causal)
    for meta in _metas():
        rows = np.arange(len(meta.view.lengths), dtype=np.int32) * 3
        n_items, max_run, plan, gen = _prefill_plan_meta(meta, cfg, rows, 1)
        runs = suffix_runs(meta)
        if runs is None:
            assert n_items == -1
            continue
        assert max_run == int(runs[1].max(initial=0))
        if max_run == 0:
            assert n_items == 0
            continue
        want = _lib.prefill_plan(runs[0], runs[1], meta.view.lengths, rows, 8, 2, causal)
        assert np.array_equal(plan.reshape(-1, _lib.PREFILL_ITEM_INTS), want)
        # the same metadata again: memo hit, same generation, same plan
        n2, _, plan2, gen2 = _prefill_plan_meta(meta, cfg, rows, 1)
        assert gen2 == gen and n2 == n_items and np.array_equal(plan2, plan)
        # below the build threshold: route known, nothing planned
        n3, m3, _, _ = _prefill_plan_meta(meta, cfg, rows, max_run + 1)
        assert n3 == 0 and m3 == max_run
