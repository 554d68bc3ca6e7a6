"""pagedkv.pool (reference pool.py) — the native allocator is host-side
already, so the drop-in pool is the engine's PagePool unchanged."""

from ..pool import MAX_POOL_PAGES, BlockTable, PageAddress, PagePool, PoolCensus  # noqa: F401
