"""pagedkv.verify (reference verify.py:1-612): the self-test suites on the
device engine, with numpy-returning attention instances."""

from __future__ import annotations

from .. import verify as _v
from ..verify import (  # noqa: F401
    HEAD_COUNT_GRID,
    HEAD_DIM_GRID,
    ORACLE_REL_TOL,
    PAGE_SIZE_GRID,
    MirrorStore,
    ScriptResult,
    VerifyCheck,
    VerifyResult,
    main,
    relative_error,
    run_allocator_script,
    run_fork_isolation,
    run_verification,
)
from .attention import gathered_attention, paged_attention, reference_attention
from .store import KvStore


class AttentionInstance(_v.AttentionInstance):
    """verify.py:110-139 — outputs are numpy."""

    def paged_output(self, stats=None, **kw):
        return paged_attention(self.queries, self.store, self.meta, self.config, stats=stats, **kw)

    def gathered_output(self, **kw):
        k, v = self.store.gather_view(self.meta.view)
        return gathered_attention(self.queries, k, v, self.meta, self.config, **kw)

    def reference_output(self):
        return reference_attention(self.queries, self.keys, self.values, self.lengths, causal=self.config.causal,
                                   scale=self.config.scale, q_lengths=self.q_lengths)


def build_attention_instance(rng, lengths, *, head_count, head_dim, page_size, causal, q_lengths=None,
                             scatter=True, device=None):
    """verify.py:142-212: same seeded draw as the reference."""
    return _v.build_attention_instance(rng, lengths, head_count=head_count, head_dim=head_dim,
                                       page_size=page_size, causal=causal, q_lengths=q_lengths, scatter=scatter,
                                       device=device, _store_cls=KvStore, _instance_cls=AttentionInstance)


def sample_attention_instance(rng, **kw):
    """verify.py:215-255 with numpy-returning instances."""
    return _v.sample_attention_instance(rng, _store_cls=KvStore, _instance_cls=AttentionInstance, **kw)
