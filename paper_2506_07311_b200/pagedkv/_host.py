"""Host (numpy) views of device tensors for the drop-in namespace."""

from __future__ import annotations

import numpy as np


def to_numpy(x):
    """torch tensor (any device) -> numpy; bf16 widens to float32 (numpy has
    no bfloat16).  numpy input passes through."""
    import torch

    if isinstance(x, torch.Tensor):
        x = x.detach()
        if x.dtype == torch.bfloat16:
            x = x.float()
        return x.cpu().numpy()
    return x


def _index(idx, device):
    import torch

    if isinstance(idx, tuple):
        return tuple(_index(i, device) for i in idx)
    if isinstance(idx, (list, np.ndarray)):
        arr = np.asarray(idx)
        return torch.from_numpy(arr.astype(np.int64) if arr.dtype != np.bool_ else arr).to(device)
    if isinstance(idx, np.integer):
        return int(idx)
    return idx


class HostRows:
    """numpy-facing view of a `[rows, heads, head_dim]` cache in HBM (the
    reference's `KvStore.keys` / `.values`, store.py:74-76).  Reads copy only
    the indexed rows to the host; writes go straight to the device."""

    __slots__ = ("_t",)

    def __init__(self, tensor):
        self._t = tensor

    @property
    def tensor(self):
        """The device tensor behind the view (the engine's fast path)."""
        return self._t

    @property
    def shape(self):
        return tuple(self._t.shape)

    @property
    def ndim(self):
        return self._t.dim()

    @property
    def size(self):
        return self._t.numel()

    @property
    def dtype(self):
        import torch

        return np.dtype(np.float32) if self._t.dtype == torch.bfloat16 else np.dtype(
            str(self._t.dtype).replace("torch.", ""))

    def __len__(self):
        return self._t.shape[0]

    def __getitem__(self, idx):
        return to_numpy(self._t[_index(idx, self._t.device)])

    def __setitem__(self, idx, value):
        import torch

        src = torch.as_tensor(np.asarray(value)).to(device=self._t.device, dtype=self._t.dtype)
        self._t[_index(idx, self._t.device)] = src

    def __array__(self, dtype=None, copy=None):
        a = to_numpy(self._t)
        return a if dtype is None else a.astype(dtype, copy=False)

    def __iter__(self):
        return iter(np.asarray(self))

    def __repr__(self):
        return f"HostRows(shape={self.shape}, dtype={self.dtype}, device={self._t.device})"
