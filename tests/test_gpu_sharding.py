"""RequestShard on one GPU: each rank's share of a request-sharded batch runs
the full decode step locally (no collective) and matches float64 on its own
sequences; together the shards cover the batch."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import relative_error  # noqa: E402
from paper_2506_07311_b200.sharding import RequestShard, lpt_partition  # noqa: E402
from replay import as_numpy  # noqa: E402

pytestmark = pytest.mark.gpu


def test_request_shards_decode_their_sequences():
    lengths = [700, 33, 1500, 16, 260, 900, 64]
    world, hq, hkv, d, ps = 2, 16, 4, 128, 16
    covered = []
    for rank in range(world):
        sh = RequestShard(lengths, rank=rank, world=world, hq=hq, hkv=hkv, head_dim=d, page_size=ps,
                          dtype=torch.bfloat16, device="cuda", headroom_tokens=4)
        assert sh.indices == lpt_partition(lengths, world)[rank]
        covered += sh.indices
        store = sh.stores[0]
        gen = torch.Generator(device="cuda").manual_seed(rank)
        ks, vs = [], []
        for s, n in zip(sh.seq_ids, sh.lengths):
            k = torch.randn((n, hkv, d), generator=gen, device="cuda").bfloat16()
            v = torch.randn((n, hkv, d), generator=gen, device="cuda").bfloat16()
            store.assign(s, np.arange(n), k, v)
            ks.append(k)
            vs.append(v)
        B = len(sh.seq_ids)
        q = torch.randn((B, hq, d), generator=gen, device="cuda").bfloat16()
        kn = torch.randn((B, hkv, d), generator=gen, device="cuda").bfloat16()
        vn = torch.randn((B, hkv, d), generator=gen, device="cuda").bfloat16()
        out = sh.step(q, kn, vn)
        for b in range(B):  # the new token is appended, then attended
            k = torch.cat([ks[b], kn[b:b + 1]]).double().repeat_interleave(hq // hkv, 1)
            v = torch.cat([vs[b], vn[b:b + 1]]).double().repeat_interleave(hq // hkv, 1)
            p = torch.softmax(torch.einsum("hd,lhd->hl", q[b].double(), k) * sh.config.scale, -1)
            ref = torch.einsum("hl,lhd->hd", p, v)
            assert relative_error(as_numpy(out[b]), ref.cpu().numpy()) <= 6e-3
        rep = sh.kv_report()
        assert rep["tokens"] == sum(n + 1 for n in sh.lengths)
        assert rep["overhead"] < 0.5
    assert sorted(covered) == list(range(len(lengths)))


def test_head_shards_reassemble_the_full_decode():
    """Head-sharded mode (§8 e-2) simulated on one GPU: the two ranks' head
    slices, concatenated in rank order (what head_shard_gather does over
    NCCL), match a float64 reference of the full-width decode."""
    from paper_2506_07311_b200.sharding import HeadShard

    lengths = [300, 17, 1200]
    world, hq, hkv, d, ps = 2, 32, 8, 128, 16
    gen = torch.Generator(device="cuda").manual_seed(9)
    ks = [torch.randn((n + 1, hkv, d), generator=gen, device="cuda").bfloat16() for n in lengths]
    vs = [torch.randn((n + 1, hkv, d), generator=gen, device="cuda").bfloat16() for n in lengths]
    q = torch.randn((len(lengths), hq, d), generator=gen, device="cuda").bfloat16()
    kn = torch.stack([k[-1] for k in ks])
    vn = torch.stack([v[-1] for v in vs])
    outs, dumps = [], []
    for rank in range(world):
        sh = HeadShard(lengths, rank=rank, world=world, hq=hq, hkv=hkv, head_dim=d, page_size=ps,
                       dtype=torch.bfloat16, device="cuda", headroom_tokens=4)
        for s, n in enumerate(lengths):
            sh.assign(s, np.arange(n), ks[s][:n], vs[s][:n])
        outs.append(sh.step(q, kn, vn))  # no process group: the local slice
        dumps.append(sh.pool.dump())
    assert dumps[0] == dumps[1]  # replicated allocator: identical tables on every rank
    full = torch.cat(outs, dim=1)
    for b in range(len(lengths)):
        k = ks[b].double().repeat_interleave(hq // hkv, 1)
        v = vs[b].double().repeat_interleave(hq // hkv, 1)
        p = torch.softmax(torch.einsum("hd,lhd->hl", q[b].double(), k) / np.sqrt(d), -1)
        ref = torch.einsum("hl,lhd->hd", p, v)
        assert relative_error(as_numpy(full[b]), ref.cpu().numpy()) <= 6e-3
