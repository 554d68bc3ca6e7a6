"""CPU oracle for the paged-attention hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain NumPy, the reference `pagedkv` algorithms that
the B200 engine replaces (reference tree: `pkg/src/pagedkv/`).  It is the
checker, never the thing measured or shipped:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
  `--impl reference` leg may import it;
* the product package `paper_2506_07311_b200` never imports it and has no CPU
  fallback.

Parity pinning: the restatement is checked against golden vectors produced by
running the real reference (`tests/golden/make_golden.py`, committed with its
outputs) and, when `/root/reference` is mounted, against the live reference.

Modules
-------
pool       PagePool restatement (pool.py:88-349), bit-exact allocator state
store      KvStore restatement (store.py:61-202), BatchView (store.py:22-58)
attention  MaskMeta (attention.py:51-110), streaming tile kernel
           (attention.py:171-329), float64 dense oracle (attention.py:389-447)
workloads  seeded generators for BASELINE.json configs C1-C5 and the
           scattered-page recipe of verify.py:142-212
"""

from .errors import (  # noqa: F401
    CapacityExhausted,
    DuplicateSequence,
    InvalidPrefix,
    NoAllowedKeys,
    OutOfRange,
    PagedKvError,
    ShapeMismatch,
    UnknownSequence,
)
from .pool import OraclePool  # noqa: F401
from .store import OracleBatchView, OracleStore  # noqa: F401
from .attention import (  # noqa: F401
    OracleMeta,
    dense_attention_f64,
    fold_gqa_queries,
    relative_error,
    round_bf16,
    streaming_attention,
    unfold_gqa_output,
)
