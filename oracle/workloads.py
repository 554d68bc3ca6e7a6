"""Seeded workloads shared by the oracle, the tests and the benchmark
(TEST INFRASTRUCTURE).

* `scattered_instance` restates the scattered-page recipe of the reference's
  `build_attention_instance` (verify.py:142-212): throw-away reservations
  interleaved with the real ones and then freed, so real block tables point at
  shuffled physical pages; K/V written in a random permutation order.  It is
  written against a duck-typed pool/store pair so the *same* random stream
  drives the oracle and the engine under test.
* `config_lengths` gives the context lengths of BASELINE.json configs C1-C5
  exactly as SURVEY.md §8 d-3 defines them.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Instance:
    pool: object
    store: object
    lengths: list
    q_lengths: list
    keys: np.ndarray     # contiguous originals, [sum(lengths), Hkv, D]
    values: np.ndarray
    queries: np.ndarray  # [sum(q_lengths), Hq, D]
    seq_ids: list


def scattered_instance(rng, lengths, *, kv_heads, q_heads=None, head_dim, page_size,
                       q_lengths=None, scatter=True, make_pool, make_store,
                       cast=None) -> Instance:
    """verify.py:159-212 recipe; `make_pool(capacity, page_size)` and
    `make_store(pool, heads, dim)` build the implementation under test and
    `cast` (optional) maps the fp32 K/V/Q arrays before use (e.g. bf16
    rounding)."""
    q_heads = kv_heads if q_heads is None else q_heads
    lengths = [int(n) for n in lengths]
    q_lengths = list(lengths) if q_lengths is None else [int(n) for n in q_lengths]
    total = sum(lengths)
    need = sum(-(-n // page_size) for n in lengths)
    dummy = int(rng.integers(1, need + 2)) if scatter else 0
    pool = make_pool(need + dummy + 2, page_size)
    store = make_store(pool, kv_heads, head_dim)
    keys = rng.standard_normal((total, kv_heads, head_dim)).astype(np.float32)
    values = rng.standard_normal((total, kv_heads, head_dim)).astype(np.float32)
    if cast is not None:
        keys, values = cast(keys), cast(values)
    pads = []
    left = dummy
    if scatter:
        for i in range(len(lengths)):
            if left > 0:
                take = int(rng.integers(1, left + 1))
                pool.reserve(f"_pad{i}", take * page_size)
                pads.append(f"_pad{i}")
                left -= take
    off = 0
    ids = []
    for i, n in enumerate(lengths):
        sid = f"s{i}"
        ids.append(sid)
        pool.reserve(sid, n)
        perm = rng.permutation(n)
        store.assign(sid, np.arange(n)[perm], keys[off:off + n][perm], values[off:off + n][perm])
        off += n
    for p in pads:
        pool.free(p)
    queries = rng.standard_normal((sum(q_lengths), q_heads, head_dim)).astype(np.float32)
    if cast is not None:
        queries = cast(queries)
    return Instance(pool, store, lengths, q_lengths, keys, values, queries, ids)


# ---- BASELINE.json configs ------------------------------

def config_lengths(name: str, *, batch: int | None = None, context: int | None = None) -> list:
    """Context lengths of one decode step for a named config."""
    if name == "c1":
        return [512]
    if name == "c2":
        rng = np.random.default_rng(0)
        return [int(x) for x in rng.integers(128, 2049, 32)]
    if name == "c3":
        return [int(context or 2048)] * int(batch or 1)
    if name == "c5":
        rng = np.random.default_rng(0)
        return [int(x) for x in np.exp(rng.uniform(math.log(128), math.log(32768), 512)).astype(int)]
    raise ValueError(f"unknown config {name}")


CONFIG_SHAPES = {
    # name: (q_heads, kv_heads, head_dim, page_size, dtype)
    "c1": (8, 8, 64, 16, "fp32"),
    "c2": (32, 32, 128, 16, "bf16"),
    "c3": (32, 8, 128, 16, "bf16"),
    "c4": (32, 8, 128, 16, "bf16"),
    "c5": (32, 8, 128, 16, "bf16"),
}


def lpt_partition(lengths, n_parts: int) -> list:
    """Longest-processing-time-first assignment of sequences to shards
    (SURVEY.md §8 e-1).  Ties go to the lowest shard index; returns a list of
    index lists, each in ascending sequence order."""
    order = sorted(range(len(lengths)), key=lambda i: (-int(lengths[i]), i))
    load = [0] * n_parts
    parts = [[] for _ in range(n_parts)]
    for i in order:
        j = min(range(n_parts), key=lambda p: (load[p], p))
        parts[j].append(i)
        load[j] += int(lengths[i])
    return [sorted(p) for p in parts]
