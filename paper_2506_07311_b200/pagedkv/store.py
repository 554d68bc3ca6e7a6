"""pagedkv.store (reference store.py:22-202) with numpy at the boundary."""

from __future__ import annotations

from ..store import BatchView  # noqa: F401
from ..store import KvStore as _DeviceKvStore
from ._host import HostRows, to_numpy


class KvStore(_DeviceKvStore):
    """The engine's KvStore (K/V in HBM, K1/K0 kernels) whose public arrays
    and gathers are numpy, as in the reference."""

    @property
    def keys(self) -> HostRows:
        return HostRows(self.k_cache)

    @property
    def values(self) -> HostRows:
        return HostRows(self.v_cache)

    def gather(self, seq_id, length: int):
        k, v = super().gather(seq_id, length)
        return to_numpy(k), to_numpy(v)

    def gather_view(self, view):
        k, v = super().gather_view(view)
        return to_numpy(k), to_numpy(v)
