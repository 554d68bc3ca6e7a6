"""K3 tcgen05 prefill (csrc/prefill_sm100.cu) against float64 references.

Reference semantics: _streaming_attention under MaskMeta.self_attention /
.suffix (reference attention.py:81-110, 259-329): query i of sequence s at
position q_pos attends keys [0, q_pos] of s (causal) or [0, len) (not).  The
reference has no bf16 and no GQA; bf16 parity is the north star's 2e-2
relative bar under the reference metric (verify.py:40-43), GQA follows the
query-fold restatement, checked here both against a torch
float64 dense reference and against the oracle's streaming restatement.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import OracleMeta, relative_error  # noqa: E402
from oracle.attention import fold_gqa_meta, fold_gqa_queries, streaming_attention, unfold_gqa_output  # noqa: E402
from oracle.store import OracleBatchView  # noqa: E402
from paper_2506_07311_b200 import (  # noqa: E402
    AttentionConfig,
    ConfigError,
    KvStore,
    MaskMeta,
    PagePool,
    gathered_attention,
    paged_attention,
)
from paper_2506_07311_b200.attention import suffix_runs  # noqa: E402
from replay import as_numpy  # noqa: E402

pytestmark = pytest.mark.gpu
BF16_TOL = 2e-2


def build(lengths, hkv, d, ps, dtype, seed=0, scatter=True):
    pool = PagePool(sum(-(-n // ps) + 1 + i % 3 for i, n in enumerate(lengths)) + 8, page_size=ps)
    store = KvStore(pool, hkv, d, dtype=dtype)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    ks, vs = [], []
    for i, n in enumerate(lengths):
        if scatter:
            pool.reserve(("pad", i), ps * (1 + i % 3))
        pool.reserve(i, n)
        k = torch.randn((n, hkv, d), generator=gen, device="cuda").to(store.torch_dtype)
        v = torch.randn((n, hkv, d), generator=gen, device="cuda").to(store.torch_dtype)
        store.assign(i, np.arange(n), k, v)
        ks.append(k)
        vs.append(v)
    if scatter:
        for i in range(len(lengths)):
            pool.free(("pad", i))
    return pool, store, ks, vs


def dense_prefill_f64(q, ks, vs, lengths, q_lens, g, scale, causal=True, rows=None):
    """float64 reference on the GPU; q [sum q_lens, Hq, D] sequence-major."""
    outs = []
    off = 0
    for k, v, n, ql in zip(ks, vs, lengths, q_lens):
        qq = q[off:off + ql].double()
        kk = k.double().repeat_interleave(g, dim=1)
        vv = v.double().repeat_interleave(g, dim=1)
        pos = torch.arange(n - ql, n, device=q.device)
        sel = slice(None) if rows is None else rows
        s = torch.einsum("qhd,khd->hqk", qq[sel], kk) * scale
        if causal:
            keyi = torch.arange(n, device=q.device)
            mask = keyi[None, :] > pos[sel][:, None]
            s = s.masked_fill(mask[None], float("-inf"))
        outs.append(torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), vv))
        off += ql
    return torch.cat(outs)


@pytest.mark.parametrize("hq,hkv,d", [(32, 8, 128), (8, 8, 64), (16, 2, 128), (4, 1, 64), (32, 32, 128)])
@pytest.mark.parametrize("ps", [8, 16, 64, 256])
def test_self_attention_prefill_matches_float64(hq, hkv, d, ps):
    lengths = [1, 37, 128, 129, 300, 700]
    pool, store, ks, vs = build(lengths, hkv, d, ps, torch.bfloat16, seed=hq + d + ps)
    cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
    meta = MaskMeta.self_attention(store.batch_view(list(range(len(lengths)))))
    assert suffix_runs(meta) is not None
    gen = torch.Generator(device="cuda").manual_seed(7)
    q = torch.randn((meta.query_count, hq, d), generator=gen, device="cuda").bfloat16()
    out = paged_attention(q, store, meta, cfg, precision="prefill")
    ref = dense_prefill_f64(q, ks, vs, lengths, lengths, hq // hkv, cfg.scale)
    err = relative_error(as_numpy(out), ref.cpu().numpy())
    assert err <= 6e-3, err


@pytest.mark.parametrize("causal", [True, False])
def test_suffix_prefill_and_non_causal(causal):
    lengths = [50, 300, 1025, 17]
    q_lens = [50, 200, 1000, 1]
    pool, store, ks, vs = build(lengths, 8, 128, 16, torch.bfloat16, seed=3)
    cfg = AttentionConfig(head_count=32, head_dim=128, page_size=16, kv_head_count=8, causal=causal)
    meta = MaskMeta.suffix(store.batch_view(list(range(len(lengths)))), q_lens)
    q = torch.randn((meta.query_count, 32, 128), device="cuda").bfloat16()
    out = paged_attention(q, store, meta, cfg)  # auto: runs >= 16 -> K3
    ref = dense_prefill_f64(q, ks, vs, lengths, q_lens, 4, cfg.scale, causal=causal)
    assert relative_error(as_numpy(out), ref.cpu().numpy()) <= 6e-3
    exact = paged_attention(q, store, meta, cfg, precision="exact")
    assert relative_error(as_numpy(out), as_numpy(exact)) <= BF16_TOL


def test_fp16_cache_and_16_bit_output():
    lengths = [260, 90]
    pool, store, ks, vs = build(lengths, 4, 64, 32, torch.float16, seed=11)
    cfg = AttentionConfig(head_count=16, head_dim=64, page_size=32, kv_head_count=4)
    meta = MaskMeta.self_attention(store.batch_view([0, 1]))
    q = torch.randn((meta.query_count, 16, 64), device="cuda").half()
    ref = dense_prefill_f64(q, ks, vs, lengths, lengths, 4, cfg.scale).cpu().numpy()
    out = paged_attention(q, store, meta, cfg, precision="tensor")
    assert out.dtype == torch.float32
    assert relative_error(as_numpy(out), ref) <= 2e-3
    out16 = paged_attention(q, store, meta, cfg, precision="tensor", out_dtype=torch.float16)
    assert out16.dtype == torch.float16
    assert relative_error(as_numpy(out16), ref) <= 4e-3


def test_paged_equals_gathered_bitwise_and_deterministic():
    lengths = [40, 130, 300]
    pool, store, ks, vs = build(lengths, 2, 128, 16, torch.bfloat16)
    cfg = AttentionConfig(head_count=8, head_dim=128, page_size=16, kv_head_count=2)
    view = store.batch_view(list(range(3)))
    meta = MaskMeta.self_attention(view)
    q = torch.randn((meta.query_count, 8, 128), device="cuda").bfloat16()
    paged = paged_attention(q, store, meta, cfg)
    gk, gv = store.gather_view(view)
    assert torch.equal(paged, gathered_attention(q, gk, gv, meta, cfg))
    assert torch.equal(paged, paged_attention(q, store, meta, cfg))


def test_matches_oracle_streaming_restatement():
    """Small case through the oracle's restatement of the reference kernel
    (GQA folded onto the reference's MHA kernel)."""
    lengths = [200, 64]
    hq, hkv, d, ps = 8, 2, 64, 16
    pool, store, ks, vs = build(lengths, hkv, d, ps, torch.bfloat16, seed=21)
    cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
    meta = MaskMeta.self_attention(store.batch_view([0, 1]))
    q = torch.randn((meta.query_count, hq, d), device="cuda").bfloat16()
    out = as_numpy(paged_attention(q, store, meta, cfg, precision="prefill"))
    keys = torch.cat(ks).float().cpu().numpy()
    vals = torch.cat(vs).float().cpu().numpy()
    ometa = OracleMeta.self_attention(OracleBatchView(lengths))
    want = unfold_gqa_output(streaming_attention(
        fold_gqa_queries(q.float().cpu().numpy(), hkv), keys, vals, fold_gqa_meta(ometa, hq // hkv),
        scale=cfg.scale, causal=True, tile=ps), hq)
    assert relative_error(out, want) <= 6e-3


@pytest.mark.parametrize("n", [2048, 8192])
def test_c4_long_prompt_rows_match_float64(n):
    """C4 shape (Llama-3-8B GQA 32q/8kv x128, one long prompt): every query
    row is computed, a spread of 96 rows is checked against float64."""
    pool, store, ks, vs = build([n], 8, 128, 16, torch.bfloat16, seed=n, scatter=True)
    cfg = AttentionConfig(head_count=32, head_dim=128, page_size=16, kv_head_count=8)
    meta = MaskMeta.self_attention(store.batch_view([0]))
    q = torch.randn((n, 32, 128), device="cuda").bfloat16()
    out = paged_attention(q, store, meta, cfg)
    assert torch.isfinite(out).all()
    rows = torch.cat([torch.arange(0, 32), torch.randint(32, n, (64,), generator=torch.Generator().manual_seed(0))]).cuda()
    ref = dense_prefill_f64(q, ks, vs, [n], [n], 4, cfg.scale, rows=rows)
    assert relative_error(as_numpy(out[rows]), ref.cpu().numpy()) <= 6e-3


def test_forced_prefill_rejects_unsupported_shapes():
    pool, store, ks, vs = build([40], 2, 64, 4, torch.bfloat16)  # page size 4 < 8
    cfg = AttentionConfig(head_count=4, head_dim=64, page_size=4, kv_head_count=2)
    meta = MaskMeta.self_attention(store.batch_view([0]))
    q = torch.randn((40, 4, 64), device="cuda").bfloat16()
    with pytest.raises(ConfigError):
        paged_attention(q, store, meta, cfg, precision="prefill")
    # auto falls back to the decode kernels for the same call
    ref = dense_prefill_f64(q, ks, vs, [40], [40], 2, cfg.scale)
    assert relative_error(as_numpy(paged_attention(q, store, meta, cfg)), ref.cpu().numpy()) <= 6e-3


@pytest.mark.parametrize("seed", range(6))
def test_random_prefill_shapes_stress(seed):
    """Random suffix metas over random batches (GQA group, head dim, page
    size, dtype, causal) through K3 against float64 on sampled rows."""
    rng = np.random.default_rng(200 + seed)
    hkv = int(rng.choice([1, 2, 4, 8]))
    g = int(rng.choice([1, 2, 4, 8, 16]))
    d = int(rng.choice([64, 128]))
    ps = int(rng.choice([8, 16, 64, 256]))
    causal = bool(seed % 3)
    dtype = torch.bfloat16 if seed % 2 == 0 else torch.float16
    lengths = [int(x) for x in rng.integers(1, 1500, int(rng.integers(1, 7)))]
    q_lens = [int(rng.integers(1, n + 1)) for n in lengths]
    pool, store, ks, vs = build(lengths, hkv, d, ps, dtype, seed=seed)
    cfg = AttentionConfig(head_count=hkv * g, head_dim=d, page_size=ps, kv_head_count=hkv, causal=causal)
    meta = MaskMeta.suffix(store.batch_view(list(range(len(lengths)))), q_lens)
    q = torch.randn((meta.query_count, hkv * g, d), device="cuda").to(dtype)
    out = paged_attention(q, store, meta, cfg, precision="prefill")
    assert torch.isfinite(out).all()
    ref = dense_prefill_f64(q, ks, vs, lengths, q_lens, g, cfg.scale, causal=causal)
    assert relative_error(as_numpy(out), ref.cpu().numpy()) <= 6e-3, seed


@pytest.mark.parametrize("ps", [8, 16, 32])
def test_fragmented_and_contiguous_page_runs_in_one_prefill(ps):
    """K3 fetches a 128-key tile whose pages form one physically contiguous
    run with one 128-row TMA box per chunk, other tiles page by page.  Build
    sequences whose first pages are interleaved with other allocations
    (fragmented tiles) and whose later pages are contiguous (run tiles), plus
    a fully permuted one: paged == gathered bitwise, and float64 parity."""
    rng = np.random.default_rng(ps)
    lengths = [1000, 777, 300]
    hq, hkv, d = 32, 8, 128
    total = sum(-(-n // ps) for n in lengths)
    pool = PagePool(3 * total + 64, page_size=ps)
    store = KvStore(pool, hkv, d, dtype=torch.bfloat16)
    pads = []
    for i, n in enumerate(lengths):
        pool.reserve(i, 0)
    # sequences 0 and 1: the first half of their pages interleaved with pads
    for t in range(-(-max(lengths[:2]) // ps) // 2):
        for i in (0, 1):
            pool.grow(i, min(lengths[i], (t + 1) * ps))
            pads.append(("pad", i, t))
            pool.reserve(pads[-1], ps)
    for i in (0, 1):
        pool.grow(i, lengths[i])  # the rest contiguous
    # sequence 2: pages drawn from a shuffled free list
    junk = [("junk", j) for j in range(-(-lengths[2] // ps) + 4)]
    for j in junk:
        pool.reserve(j, ps)
    for j in rng.permutation(len(junk)):
        pool.free(junk[j])
    pool.grow(2, lengths[2])
    for pd in pads:
        pool.free(pd)
    entries = [np.asarray(pool.table(i).entries) for i in range(3)]
    assert any((np.diff(e) != 1).any() for e in entries)  # some tiles are fragmented
    gen = torch.Generator(device="cuda").manual_seed(ps)
    ks, vs = [], []
    for i, n in enumerate(lengths):
        pool.table(i).logical_len = 0
        k = torch.randn((n, hkv, d), generator=gen, device="cuda").bfloat16()
        v = torch.randn((n, hkv, d), generator=gen, device="cuda").bfloat16()
        store.assign(i, np.arange(n), k, v)
        ks.append(k)
        vs.append(v)
    cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
    view = store.batch_view([0, 1, 2])
    meta = MaskMeta.self_attention(view)
    q = torch.randn((meta.query_count, hq, d), generator=gen, device="cuda").bfloat16()
    paged = paged_attention(q, store, meta, cfg, precision="prefill")
    gk, gv = store.gather_view(view)
    assert torch.equal(paged, gathered_attention(q, gk, gv, meta, cfg, precision="prefill"))
    ref = dense_prefill_f64(q, ks, vs, lengths, lengths, hq // hkv, cfg.scale)
    assert relative_error(as_numpy(paged), ref.cpu().numpy()) <= 6e-3


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d", [64, 128])
def test_tma_store_and_register_store_epilogues(out_dtype, d):
    """Full query tiles leave K3 by TMA stores staged in shared memory,
    partial tiles (a prompt length that is not a multiple of the tile) by
    register stores: both, in fp32 and bf16 output, against float64."""
    lengths = [700, 333, 64]  # 700 / 32 and 333 / 32 leave partial tiles (G = 4: 32 positions per tile)
    pool, store, ks, vs = build(lengths, 8, d, 16, torch.bfloat16, seed=d)
    cfg = AttentionConfig(head_count=32, head_dim=d, page_size=16, kv_head_count=8)
    meta = MaskMeta.self_attention(store.batch_view([0, 1, 2]))
    gen = torch.Generator(device="cuda").manual_seed(d)
    q = torch.randn((meta.query_count, 32, d), generator=gen, device="cuda").bfloat16()
    out = paged_attention(q, store, meta, cfg, precision="prefill", out_dtype=out_dtype)
    assert out.dtype == out_dtype
    ref = dense_prefill_f64(q, ks, vs, lengths, lengths, 4, cfg.scale)
    assert relative_error(as_numpy(out.float()), ref.cpu().numpy()) <= (6e-3 if out_dtype == torch.float32 else 1e-2)


def test_repeat_call_fast_path_and_its_invalidation(monkeypatch):
    """paged_attention's repeat-call path (attention._prefill_fast): the same
    sealed meta / store / config again relaunches the prepared K3 argument
    block — bitwise the full path's result, new q / out pointers honoured —
    and any pool change, another plan in this thread's device buffer, a
    corrupted view or an unsealed meta falls back to the full path."""
    from paper_2506_07311_b200 import attention as A
    from paper_2506_07311_b200.errors import NoAllowedKeys

    hq, hkv, d, ps = 8, 2, 128, 16
    lengths = [300, 129]
    pool, store, ks, vs = build(lengths, hkv, d, ps, torch.bfloat16, seed=11)
    cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
    meta = MaskMeta.self_attention(store.batch_view([0, 1]))
    assert not meta.q_seq.flags.writeable and not meta.q_pos.flags.writeable
    gen = torch.Generator(device="cuda").manual_seed(3)
    qs = [torch.randn((sum(lengths), hq, d), generator=gen, device="cuda").bfloat16() for _ in range(2)]
    full = [paged_attention(q, store, meta, cfg).clone() for q in qs]  # second call may already be fast

    calls = {"route": 0}
    real_route = A._prefill_route

    def counting_route(*a, **k):
        calls["route"] += 1
        return real_route(*a, **k)

    monkeypatch.setattr(A, "_prefill_route", counting_route)
    for i in range(4):  # alternate q tensors: every call on the fast path, each with its own q
        out = paged_attention(qs[i % 2], store, meta, cfg)
        assert torch.equal(out, full[i % 2])
    assert calls["route"] == 0

    # another meta's plan replaces this thread's device plan: full path, same result
    other = MaskMeta.suffix(store.batch_view([0]), [40])
    paged_attention(qs[0][:40], store, other, cfg)
    before = calls["route"]
    assert torch.equal(paged_attention(qs[0], store, meta, cfg), full[0])
    assert calls["route"] == before + 1
    assert torch.equal(paged_attention(qs[1], store, meta, cfg), full[1])
    assert calls["route"] == before + 1  # fast again

    # a pool mutation (unrelated sequence) bumps the generation: full path once
    pool.reserve("other", 40)
    assert torch.equal(paged_attention(qs[0], store, meta, cfg), full[0])
    assert calls["route"] == before + 2
    # the output dtype is part of the key
    o16 = paged_attention(qs[0], store, meta, cfg, out_dtype=torch.bfloat16)
    assert o16.dtype == torch.bfloat16 and calls["route"] == before + 3

    # an unsealed meta with equal content never takes the fast path
    loose = MaskMeta(view=meta.view, q_seq=meta.q_seq.copy(), q_pos=meta.q_pos.copy())
    paged_attention(qs[0], store, loose, cfg)
    paged_attention(qs[0], store, loose, cfg)
    assert calls["route"] == before + 5

    # corrupting the view in place (the reference suite does this) is seen
    paged_attention(qs[0], store, meta, cfg)
    meta.view.lengths[1] = 0
    with pytest.raises((NoAllowedKeys, Exception)):
        paged_attention(qs[0], store, meta, cfg)
    meta.view.lengths[1] = lengths[1]
