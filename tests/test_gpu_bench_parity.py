"""Parity of the exact configurations bench.py times.

bench.DecodeBench is the object bench.py times: one pkv_paged_attention call
per step with the K1 append fused and the host plan precomputed.  Here it is
driven for a few steps and checked

* C2 (MHA 32x128 bf16, batch 32, contexts 128-2048): against the CPU oracle
  (float64 dense attention over the sequence's K/V read back from its pages)
  on every sequence, and through DecodeBench.verify (the check bench.py
  itself reports as `parity_checked`);
* C5 at full size (512 sequences, log-uniform 128-32k, 14 GB of KV, the
  capped 128-CTA grid with cut units): through DecodeBench.verify on 48
  sampled sequences, the appended rows of every step bit-exact;
* both on a fragmented pool (random page permutation).

References: attention.py:259-329 (the streaming kernel), store.py:146-150
(the scatter of the appended rows).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import bench  # noqa: E402
from oracle import dense_attention_f64, relative_error  # noqa: E402

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def _bench(config, steps, fragment=False, e2e_steps=None):
    _, lengths, hq, hkv, d, ps = bench.workload(config, 0, 1)
    dev = torch.device("cuda", 0)
    b = bench.DecodeBench(lengths, hq, hkv, d, ps, total_steps=steps, device=dev, seed=0, fragment=fragment,
                          e2e_steps=e2e_steps)
    for t in range(steps):
        b.step(t)
    torch.cuda.synchronize()
    return b


@pytest.mark.parametrize("fragment", [False, True])
def test_c2_exact_bench_call_against_oracle(fragment):
    steps = 3
    b = _bench("c2", steps, fragment)
    assert (b.hq, b.hkv, b.d, b.ps, b.B) == (32, 32, 128, 16, 32)
    out = b.out.cpu().numpy()
    t = steps - 1
    ks, vs, qs = [], [], b.qs[t].float().cpu().numpy()
    lens = []
    for s in range(b.B):
        L = b.lengths[s] + steps
        entries = np.asarray(list(b.pool.table(s).entries), dtype=np.int64)
        pos = np.arange(L)
        rows = torch.from_numpy(entries[pos // 16] * 16 + pos % 16).cuda()
        k = b.store.k_cache.index_select(0, rows)
        v = b.store.v_cache.index_select(0, rows)
        # the fused append wrote every step's token into its page, bit-exact
        assert torch.equal(k[b.lengths[s]:], b.ks[:steps, s])
        assert torch.equal(v[b.lengths[s]:], b.vs[:steps, s])
        ks.append(k.float().cpu().numpy())
        vs.append(v.float().cpu().numpy())
        lens.append(L)
    ref = dense_attention_f64(qs, np.concatenate(ks), np.concatenate(vs), lens, causal=True,
                              q_lengths=[1] * b.B)
    assert relative_error(out, ref) <= BF16_TOL
    v = b.verify(n_sample=32)
    assert v["ok"] and v["sequences"] == 32 and v["appended_rows_bit_exact"], v


@pytest.mark.parametrize("fragment", [False, True])
def test_c5_full_size_exact_bench_call(fragment):
    steps = 2
    b = _bench("c5", steps, fragment)
    assert b.B == 512 and sum(b.lengths) == 3_431_895
    v = b.verify(n_sample=48, seed=1)
    assert v["ok"] and v["sequences"] == 48, v
    # the longest and the shortest sequences are always among the checked ones
    v2 = b.verify(n_sample=2, seed=2)
    assert v2["ok"], v2
    order = np.argsort(b.lengths)
    for idx in (order[0], order[-1]):
        b_idx = int(idx)
        L = b.lengths[b_idx] + steps
        entries = np.asarray(list(b.pool.table(b_idx).entries), dtype=np.int64)
        pos = np.arange(L)
        rows = torch.from_numpy(entries[pos // 16] * 16 + pos % 16).cuda()
        k = b.store.k_cache.index_select(0, rows).double().repeat_interleave(4, dim=1)
        vv = b.store.v_cache.index_select(0, rows).double().repeat_interleave(4, dim=1)
        q = b.qs[steps - 1, b_idx].double()
        p = torch.softmax(torch.einsum("hd,khd->hk", q, k) * b.cfg.scale, dim=-1)
        ref = torch.einsum("hk,khd->hd", p, vv)
        err = float((b.out[b_idx].double() - ref).abs().max() / ref.abs().max())
        assert err <= BF16_TOL, (b_idx, L, err)


def _f64_decode(b, s, q, L):
    entries = np.asarray(list(b.pool.table(s).entries), dtype=np.int64)
    pos = np.arange(L)
    rows = torch.from_numpy(entries[pos // b.ps] * b.ps + pos % b.ps).cuda()
    g = b.hq // b.hkv
    k = b.store.k_cache.index_select(0, rows).double().repeat_interleave(g, dim=1)
    v = b.store.v_cache.index_select(0, rows).double().repeat_interleave(g, dim=1)
    p = torch.softmax(torch.einsum("hd,khd->hk", q.double().cuda(), k) * b.cfg.scale, dim=-1)
    return torch.einsum("hk,khd->hd", p, v)


def test_bench_e2e_path_grants_pages_and_stays_correct():
    """The e2e leg (DecodeBatch.step after the device phase) continues the
    sequences from the device phase's tokens, takes page grants from the
    allocator, and the next API step is still correct."""
    from paper_2506_07311_b200.batch import DecodeBatch

    steps = 2
    b = _bench("c2", steps, e2e_steps=24)
    e = b.run_e2e(1, 20, lambda: None)
    assert e["pages_granted"] > 0
    for s in range(b.B):
        assert b.pool.table(s).logical_len == b.lengths[s] + steps + 21
    g = torch.Generator().manual_seed(5)
    q = torch.randn((b.B, b.hq, b.d), generator=g).bfloat16()
    k = torch.randn((b.B, b.hkv, b.d), generator=g).bfloat16()
    v = torch.randn((b.B, b.hkv, b.d), generator=g).bfloat16()
    out = DecodeBatch(b.store, list(range(b.B)), b.cfg).step(q, k, v)
    torch.cuda.synchronize()
    for s in range(b.B):
        L = b.pool.table(s).logical_len
        ref = _f64_decode(b, s, q[s].float(), L)
        assert float((out[s].double() - ref).abs().max() / ref.abs().max()) <= BF16_TOL
