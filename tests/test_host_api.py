"""Host-side API of the drop-in (no GPU): the reference's own known-answer
tests for the batch view, mask metadata and block classification, ported to
the package (reference tests/test_store.py:172-189, tests/test_attention.py:
63-124).  The device kernels never see the block mask; it backs KernelStats
parity (attention.py:213-226)."""

import numpy as np
import pytest

from paper_2506_07311_b200 import (
    AttentionConfig,
    BatchView,
    BlockKind,
    MaskMeta,
    OutOfRange,
    ShapeMismatch,
    build_block_mask,
    mask_allow,
)


def small_meta(lengths):
    return MaskMeta.self_attention(BatchView.from_lengths(lengths))


def test_batch_view_layout():
    view = BatchView.from_lengths([3, 2], ids=["a", "b"])
    assert view.prefix_sums.tolist() == [0, 3]
    assert view.slot_seq.tolist() == [0, 0, 0, 1, 1]
    assert view.slot_local.tolist() == [0, 1, 2, 0, 1]
    assert view.total_slots == 5
    single = BatchView.from_lengths([7])
    assert single.prefix_sums.tolist() == [0] and (single.slot_seq == 0).all()


def test_batch_view_ladder_totals():
    lengths = list(range(500, 8001, 500))
    view = BatchView.from_lengths(lengths)
    assert view.total_slots == 68000
    assert view.prefix_sums[-1] + lengths[-1] == 68000


def test_mask_meta_validation():
    view = BatchView.from_lengths([4, 4])
    with pytest.raises(ValueError):
        MaskMeta(view=view, q_seq=np.array([1, 0]), q_pos=np.array([0, 0]))  # not sequence-major
    with pytest.raises(OutOfRange):
        MaskMeta(view=view, q_seq=np.array([0]), q_pos=np.array([4]))
    with pytest.raises(ShapeMismatch):
        MaskMeta(view=view, q_seq=np.array([0, 1]), q_pos=np.array([0]))
    with pytest.raises(OutOfRange):
        MaskMeta.decode(BatchView.from_lengths([3, 0]))
    m = MaskMeta.suffix(view, [1, 2])
    assert m.q_seq.tolist() == [0, 1, 1] and m.q_pos.tolist() == [3, 2, 3]


def test_block_mask_two_sequences_block_aligned_noncausal():
    cfg = AttentionConfig(head_count=1, head_dim=8, causal=False, page_size=16)
    mask = build_block_mask(small_meta([32, 32]), cfg)
    expected = np.array([[2, 2, 0, 0], [2, 2, 0, 0], [0, 0, 2, 2], [0, 0, 2, 2]], dtype=np.int8)
    assert mask.counts()["partial"] == 0 and np.array_equal(mask.kinds, expected)


def test_block_mask_causal_lower_triangle():
    cfg = AttentionConfig(head_count=1, head_dim=8, causal=True, page_size=16)
    mask = build_block_mask(small_meta([48]), cfg)
    assert [BlockKind(k) for k in np.diag(mask.kinds)] == [BlockKind.PARTIAL] * 3
    assert mask.kind(1, 0) == BlockKind.FULL and mask.kind(2, 0) == BlockKind.FULL
    assert mask.kind(0, 1) == BlockKind.EMPTY and mask.kind(0, 2) == BlockKind.EMPTY


@pytest.mark.parametrize("seed", range(6))
def test_block_mask_matches_exhaustive_predicate(seed):
    rng = np.random.default_rng(seed)
    lengths = [int(rng.integers(1, 120)) for _ in range(int(rng.integers(1, 5)))]
    causal = bool(rng.integers(2))
    cfg = AttentionConfig(head_count=1, head_dim=8, causal=causal, page_size=16)
    meta = small_meta(lengths)
    mask = build_block_mask(meta, cfg)
    q_len, kv_len = meta.query_count, meta.view.total_slots
    for qb in range(mask.kinds.shape[0]):
        for kb in range(mask.kinds.shape[1]):
            qs = range(qb * 16, min((qb + 1) * 16, q_len))
            ks = range(kb * 16, min((kb + 1) * 16, kv_len))
            hits = sum(mask_allow(q, k, meta, causal=causal) for q in qs for k in ks)
            want = BlockKind.EMPTY if hits == 0 else BlockKind.FULL if hits == len(qs) * len(ks) else BlockKind.PARTIAL
            assert mask.kind(qb, kb) == want, (qb, kb)


def test_attention_config_defaults_and_validation():
    cfg = AttentionConfig(head_count=8, head_dim=64)
    assert cfg.scale == pytest.approx(1 / 8) and cfg.causal and cfg.page_size == 64 and cfg.kv_head_count == 8
    for bad in (dict(page_size=48), dict(scale=-1.0), dict(kv_head_count=3)):
        with pytest.raises(ValueError):
            AttentionConfig(head_count=8, head_dim=64, **bad)


def test_mask_meta_constructors_seal_their_query_arrays():
    """self_attention / decode / suffix build fresh query arrays and mark them
    read-only (the identity key of paged_attention's repeat-call path); a
    directly constructed meta keeps the caller's arrays as they are, and the
    view's lengths stay writeable (the reference suite corrupts them)."""
    view = BatchView.from_lengths([5, 3])
    for meta in (MaskMeta.self_attention(view), MaskMeta.decode(view), MaskMeta.suffix(view, [2, 1])):
        assert not meta.q_seq.flags.writeable and not meta.q_pos.flags.writeable
        with pytest.raises(ValueError):
            meta.q_pos[0] = 0
    q_seq, q_pos = np.array([0, 1]), np.array([4, 2])
    loose = MaskMeta(view=view, q_seq=q_seq, q_pos=q_pos)
    assert loose.q_seq.flags.writeable and loose.q_pos.flags.writeable
    assert view.lengths.flags.writeable
