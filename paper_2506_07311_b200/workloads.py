"""Synthetic decode workloads of BASELINE.json configs C1-C5.

Product-side generator used by bench.py and the sharder; the oracle keeps an
independent copy (oracle/workloads.py) and tests/test_sharding.py checks the
two agree.  Context lengths follow the survey exactly: C2 draws 32 lengths in
[128, 2048] from default_rng(0) (sum 36,477); C5 draws 512 log-uniform lengths
in [128, 32768] from default_rng(0) (sum 3,431,895).
"""

from __future__ import annotations

import math

import numpy as np

# name: (q_heads, kv_heads, head_dim, page_size, dtype)
CONFIG_SHAPES = {
    "c1": (8, 8, 64, 16, "fp32"),
    "c2": (32, 32, 128, 16, "bf16"),
    "c3": (32, 8, 128, 16, "bf16"),
    "c4": (32, 8, 128, 16, "bf16"),
    "c5": (32, 8, 128, 16, "bf16"),
}


def config_lengths(name: str, *, batch: int | None = None, context: int | None = None) -> list:
    """Context lengths of one decode step of a named config."""
    if name == "c1":
        return [512]
    if name == "c2":
        rng = np.random.default_rng(0)
        return [int(x) for x in rng.integers(128, 2049, 32)]
    if name == "c3":
        return [int(context or 2048)] * int(batch or 1)
    if name == "c4":
        return [int(context or 8192)] * int(batch or 1)
    if name == "c5":
        rng = np.random.default_rng(0)
        return [int(x) for x in np.exp(rng.uniform(math.log(128), math.log(32768), 512)).astype(int)]
    raise ValueError(f"unknown config {name}")
