"""FMS-style decode loop — the caller of the hot path (reference decoder.py:196-287).

`PagedDecoderCache` / `DecodeSession` keep the reference API and call order
(grow -> assign -> batch_view -> MaskMeta -> paged_attention, decoder.py:236-284)
but the cache lives in HBM and attention runs on the device.  The model object
is duck-typed on the reference's `ToyDecoder` (embed, blocks, _qkv,
_finish_block, _logits, config); the toy model itself is out of scope.
"""

from __future__ import annotations

import numpy as np

from .attention import AttentionConfig, KernelStats, MaskMeta, paged_attention
from .pool import PagePool
from .store import KvStore


def _layer_norm(x, gain, bias):
    mean = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mean) / np.sqrt(var + 1e-5) * gain + bias


class PagedDecoderCache:
    """Per-layer KV stores over one shared page pool (decoder.py:196-210)."""

    def __init__(self, decoder, pool: PagePool, dtype=np.float32, device=None):
        cfg = decoder.config
        self.pool = pool
        kv_heads = getattr(cfg, "kv_head_count", None) or cfg.head_count
        self.stores = [KvStore(pool, kv_heads, cfg.head_dim, dtype=dtype, device=device)
                       for _ in range(cfg.layers)]
        self.attn_config = AttentionConfig(head_count=cfg.head_count, head_dim=cfg.head_dim,
                                           causal=True, page_size=pool.page_size,
                                           kv_head_count=kv_heads)


class DecodeSession:
    """Cached decode of one sequence against a shared paged cache
    (decoder.py:222-287)."""

    def __init__(self, decoder, cache: PagedDecoderCache, seq_id):
        self.decoder = decoder
        self.cache = cache
        self.seq_id = seq_id
        self._len = 0
        cache.pool.reserve(seq_id, 0)

    @property
    def context_len(self) -> int:
        return self._len

    def _attend(self, store, q, meta, counter):
        stats = KernelStats()
        attn = paged_attention(q, store, meta, self.cache.attn_config, stats=stats)
        if counter:
            cfg = self.decoder.config
            counter.add_attention_pairs(stats.allowed_pairs, cfg.head_count, cfg.head_dim)
        return attn.cpu().numpy()

    def prefill(self, tokens, counter=None):
        if self._len:
            raise ValueError("prefill must happen before any decode step")
        n = len(tokens)
        if n == 0:
            raise ValueError("prompt must contain at least one token")
        dec, cache = self.decoder, self.cache
        cache.pool.grow(self.seq_id, n)
        positions = np.arange(n)
        x = dec.embed(tokens, positions)
        for store, block in zip(cache.stores, dec.blocks):
            q, k, v = dec._qkv(block, _layer_norm(x, *block["ln1"]), counter)
            store.assign(self.seq_id, positions, k, v)
            view = store.batch_view([self.seq_id])
            attn = self._attend(store, q, MaskMeta.self_attention(view), counter)
            x = dec._finish_block(block, x, attn, counter)
        self._len = n
        return dec._logits(x[-1:], counter)

    def step(self, token: int, counter=None):
        dec, cache = self.decoder, self.cache
        pos = self._len
        cache.pool.grow(self.seq_id, pos + 1)
        x = dec.embed([token], [pos])
        for store, block in zip(cache.stores, dec.blocks):
            q, k, v = dec._qkv(block, _layer_norm(x, *block["ln1"]), counter)
            store.assign(self.seq_id, [pos], k, v)
            view = store.batch_view([self.seq_id])
            attn = self._attend(store, q, MaskMeta.decode(view), counter)
            x = dec._finish_block(block, x, attn, counter)
        self._len = pos + 1
        return dec._logits(x[-1:], counter)

    def free(self) -> int:
        return self.cache.pool.free(self.seq_id)
