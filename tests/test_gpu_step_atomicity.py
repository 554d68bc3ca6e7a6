"""All-or-nothing batched decode step on the device (GPU twin of
tests/test_step_atomicity.py).

DecodeBatch.step is one native call: allocator (grow / copy-on-write /
logical_len), metadata upload, page clears, fused append + decode.  A failure
injected at the metadata upload or at the attention launch must leave the
allocator exactly as it was (dump(), refcounts) and the device mirror usable:
the retried step then produces the same caches and output as a twin batch
that never failed.  Reference contract: pool.py:143-148, 165-169.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2506_07311_b200 import AttentionConfig, DeviceError, KvStore, PagePool, _lib  # noqa: E402
from paper_2506_07311_b200.batch import DecodeBatch  # noqa: E402

pytestmark = pytest.mark.gpu


def _setup(seed):
    hq, hkv, d, ps = 8, 2, 128, 16
    pool = PagePool(256, ps)
    store = KvStore(pool, hkv, d, dtype=torch.bfloat16)
    g = torch.Generator(device="cuda").manual_seed(seed)
    lens = [16, 31, 47, 5, 64]  # 16 / 64 / 47+1 cross page boundaries on the next token
    for s, n in enumerate(lens):
        pool.reserve(s, n)
        store.assign(s, np.arange(n), torch.randn((n, hkv, d), generator=g, device="cuda").bfloat16(),
                     torch.randn((n, hkv, d), generator=g, device="cuda").bfloat16())
    pool.fork(2, "c", 32)  # the child's next token lands in a shared page -> copy-on-write
    pool.table("c").logical_len = 20
    ids = [0, 1, 2, 3, 4, "c"]
    cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
    return pool, store, DecodeBatch(store, ids, cfg), ids


def _inputs(n, seed):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn((n, 8, 128), generator=g).bfloat16(), torch.randn((n, 2, 128), generator=g).bfloat16(),
            torch.randn((n, 2, 128), generator=g).bfloat16())


def _refcounts(pool):
    return [pool.page_refcount(p) for p in range(pool.capacity_pages)]


class _Repeated:
    """A serving loop's step: the same pinned host buffers and device `out`
    every token (DecodeBatch's prepared fast path, optionally as CUDA graphs)."""

    def __init__(self, batch, n, graph):
        self.batch = batch
        batch.use_graph = graph
        self.q = torch.empty((n, 8, 128), dtype=torch.bfloat16).pin_memory()
        self.k = torch.empty((n, 2, 128), dtype=torch.bfloat16).pin_memory()
        self.v = torch.empty((n, 2, 128), dtype=torch.bfloat16).pin_memory()
        self.out = torch.empty((n, 8, 128), dtype=torch.float32, device="cuda")

    def step(self, q, k, v):
        torch.cuda.synchronize()  # the previous step has read the buffers
        self.q.copy_(q)
        self.k.copy_(k)
        self.v.copy_(v)
        return self.batch.step(self.q, self.k, self.v, out=self.out).clone()


@pytest.mark.parametrize("mode", ["call", "repeated", "graph"])
@pytest.mark.parametrize("site", [_lib.PKV_FAIL_STEP_UPLOAD, _lib.PKV_FAIL_STEP_LAUNCH])
def test_failed_step_rolls_back_and_retry_matches_twin(site, mode):
    pool_a, store_a, batch_a, ids = _setup(0)
    pool_b, store_b, batch_b, _ = _setup(0)
    step_a = batch_a.step if mode == "call" else _Repeated(batch_a, len(ids), mode == "graph").step
    for i in range(3):  # a few normal steps first (mirror and ring in use)
        q, k, v = _inputs(len(ids), i)
        step_a(q, k, v)
        batch_b.step(q, k, v)
    torch.cuda.synchronize()
    before = (pool_a.dump(), _refcounts(pool_a))
    q, k, v = _inputs(len(ids), 99)
    _lib.load().pkv_debug_inject_failure(site)
    with pytest.raises(DeviceError, match="injected"):
        step_a(q, k, v)
    torch.cuda.synchronize()
    assert (pool_a.dump(), _refcounts(pool_a)) == before
    out_a = step_a(q, k, v)
    out_b = batch_b.step(q, k, v)
    torch.cuda.synchronize()
    assert pool_a.dump() == pool_b.dump()
    assert torch.equal(out_a, out_b)
    if mode == "graph":
        assert batch_a.graph_stats()[0] >= 3  # every prepared call after the first
    for s in ids:  # the retried step wrote the same K/V into the same pages
        ka, va = store_a.gather(s, pool_a.table(s).logical_len)
        kb, vb = store_b.gather(s, pool_b.table(s).logical_len)
        assert torch.equal(ka, kb) and torch.equal(va, vb)
