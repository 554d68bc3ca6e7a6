"""numpy-facing drop-in namespace for the reference package `pagedkv`.

    import paper_2506_07311_b200.pagedkv as pagedkv

Same module layout and names as the reference (`pagedkv.errors`, `.pool`,
`.store`, `.attention`, `.verify`, `.decoder`, `.workload`; reference
__init__.py:6-59) over the same device engine, with the reference's numpy
types at the boundary:

* `KvStore.keys` / `.values` are numpy-facing views of the HBM caches
  (indexing returns numpy arrays, `np.asarray(store.keys)` copies the cache to
  the host, item assignment writes through) — reference store.py:74-76;
* `gather` / `gather_view` return numpy arrays in the store's dtype
  (store.py:152-161, 187-190);
* `paged_attention` / `gathered_attention` return float32 numpy
  (attention.py:271-272, 332-378), `reference_attention` /
  `attention_weights` float64 numpy (attention.py:389-474).

The package root (`paper_2506_07311_b200`) keeps the torch fast path: device
tensors in, device tensors out, no host round trip.  The reference's own test
suite runs unmodified against this namespace (tests/test_reference_suite.py).
Not provided: the desk-scale numpy model (decoder.py:31-194), which is not on
the paged-attention path.
"""

__version__ = "0.1.0"

from .errors import (  # noqa: F401
    CapacityExhausted,
    ConfigError,
    DuplicateSequence,
    InvalidPrefix,
    InvalidTrace,
    NoAllowedKeys,
    OutOfRange,
    PagedKvError,
    ShapeMismatch,
    UnknownSequence,
)
from .pool import BlockTable, PageAddress, PagePool, PoolCensus  # noqa: F401
from .store import BatchView, KvStore  # noqa: F401
from .attention import (  # noqa: F401
    AttentionConfig,
    BlockKind,
    BlockMask,
    KernelStats,
    MaskMeta,
    attention_weights,
    build_block_mask,
    gathered_attention,
    mask_allow,
    paged_attention,
    reference_attention,
)
from .decoder import DecodeSession, PagedDecoderCache  # noqa: F401
from .workload import (  # noqa: F401
    Arrive,
    ContiguousModel,
    Decode,
    Finish,
    ForkEvent,
    KvBytesConfig,
    MemoryReport,
    PagedModel,
    Trace,
    account,
    full_report,
    gen_chat_growth,
    gen_mixed_batch,
    gen_single_sequence,
)

SUBMODULES = ("errors", "pool", "store", "attention", "verify", "decoder", "workload")


def install_alias(name: str = "pagedkv") -> None:
    """Make `import pagedkv` (and its submodules) resolve to this namespace,
    so reference callers run unchanged."""
    import importlib
    import sys

    sys.modules[name] = sys.modules[__name__]
    for sub in SUBMODULES:
        sys.modules[f"{name}.{sub}"] = importlib.import_module(f"{__name__}.{sub}")


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("SUBMODULES", "install_alias")]
