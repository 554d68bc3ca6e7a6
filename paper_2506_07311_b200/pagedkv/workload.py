"""pagedkv.workload (reference workload.py): trace wire format, generators
and the memory audit, over the native allocator."""

from ..workload import *  # noqa: F401,F403
from ..workload import (  # noqa: F401
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
