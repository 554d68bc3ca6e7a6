"""pagedkv.attention (reference attention.py:26-474) with numpy results:
the same device kernels, outputs copied to the host."""

from __future__ import annotations

from .. import attention as _a
from ..attention import (  # noqa: F401
    AttentionConfig,
    BlockKind,
    BlockMask,
    KernelStats,
    MaskMeta,
    allowed_key_counts,
    build_block_mask,
    mask_allow,
)
from ._host import to_numpy


def _keys_arg(x):
    from ._host import HostRows

    return x.tensor if isinstance(x, HostRows) else x


def paged_attention(queries, store, meta, config, *, stats=None, block_mask=None, skip_empty=True, **kw):
    """attention.py:332-354 -> float32 numpy (n_queries, heads, head_dim)."""
    return to_numpy(_a.paged_attention(queries, store, meta, config, stats=stats, block_mask=block_mask,
                                       skip_empty=skip_empty, **kw))


def gathered_attention(queries, keys, values, meta, config, *, stats=None, block_mask=None, skip_empty=True,
                       **kw):
    """attention.py:357-378 -> float32 numpy; bitwise equal to paged_attention."""
    return to_numpy(_a.gathered_attention(queries, _keys_arg(keys), _keys_arg(values), meta, config,
                                          stats=stats, block_mask=block_mask, skip_empty=skip_empty, **kw))


def reference_attention(queries, keys, values, lengths, *, causal=True, scale=None, q_lengths=None):
    """attention.py:389-447: float64 numpy oracle (the engine computes it on
    the device in float64)."""
    return to_numpy(_a.reference_attention(queries, _keys_arg(keys), _keys_arg(values), lengths, causal=causal,
                                           scale=scale, q_lengths=q_lengths))


def attention_weights(queries, store, meta, config):
    """attention.py:450-474: float64 numpy (n_queries, heads, kv_slots)."""
    return to_numpy(_a.attention_weights(queries, store, meta, config))
