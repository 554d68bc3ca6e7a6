"""Multi-GPU request sharding (SURVEY.md §8 e) — new; the reference is single
process and lists multi-device allocation as a non-goal.

Request-sharded mode (default).  Sequences are independent, so they are
partitioned across the GPUs of one box by LPT on their context length (the
decode step's KV bytes are linear in it).  Every rank owns its own PagePool +
KvStore(s) + device block-table mirror + DecodeBatch on its own device and
runs the whole K1 -> K2 -> K2c step locally: there is no collective on the
data path.  A sequence never migrates; CapacityExhausted is per shard with
the reference's semantics, and allocator parity is per shard (replaying that
shard's op stream on a reference PagePool gives the same dump()).

Head-sharded mode (optional, §8 e-2).  Each of n ranks owns hkv/n kv heads
(and the matching hq/n query heads) of every sequence; the allocator is
replicated deterministically so block tables agree, and after the local
decode the per-rank output slices [B, hq/n, D] are all-gathered over NCCL
(NVLink/NVSwitch on a B200 box) into [B, hq, D].

KV-memory overhead uses the reference's definition (workload.py:301-349):
charged slots / theoretical minimum (a page_size = 1 pool) - 1.
"""

from __future__ import annotations

import heapq

import numpy as np


def lpt_partition(lengths, n_parts: int) -> list:
    """Longest-processing-time-first assignment of sequence indices to
    n_parts shards: sequences by descending length (ties: lower index first)
    each go to the least-loaded shard (ties: lower shard).  Returns index
    lists in ascending order.  Deterministic, so every rank computes the same
    partition without communicating."""
    if n_parts <= 0:
        raise ValueError("n_parts must be positive")
    lens = [int(x) for x in lengths]
    order = sorted(range(len(lens)), key=lambda i: (-lens[i], i))
    heap = [(0, p) for p in range(n_parts)]
    parts = [[] for _ in range(n_parts)]
    for i in order:
        load, p = heapq.heappop(heap)
        parts[p].append(i)
        heapq.heappush(heap, (load + lens[i], p))
    return [sorted(p) for p in parts]


def shard_balance(lengths, parts) -> float:
    """max shard load / mean shard load (1.0 = perfect)."""
    loads = [sum(int(lengths[i]) for i in p) for p in parts]
    mean = sum(loads) / max(len(loads), 1)
    return max(loads) / mean if mean else 1.0


def kv_overhead(lengths, page_size: int) -> dict:
    """Paged KV overhead of holding `lengths` tokens at `page_size`
    (reference workload.account: charged / theoretical minimum - 1)."""
    lens = np.asarray(lengths, dtype=np.int64)
    tokens = int(lens.sum())
    charged = int((-(-lens // page_size)).sum()) * page_size
    return {"tokens": tokens, "charged_slots": charged,
            "overhead": (charged / tokens - 1.0) if tokens else 0.0}


class RequestShard:
    """This rank's share of a request-sharded decode batch.

    `lengths` are the global batch's current context lengths (identical on
    every rank); the rank keeps the LPT part `indices` and builds its own
    pool and stores on `device`."""

    def __init__(self, lengths, *, rank: int, world: int, hq: int, hkv: int, head_dim: int,
                 page_size: int, dtype="bf16", device=None, headroom_tokens: int = 0, layers: int = 1):
        from .attention import AttentionConfig
        from .pool import PagePool
        from .store import KvStore

        self.rank, self.world = rank, world
        self.global_lengths = [int(x) for x in lengths]
        self.indices = lpt_partition(self.global_lengths, world)[rank]
        self.lengths = [self.global_lengths[i] for i in self.indices]
        pages = sum(-(-(n + headroom_tokens) // page_size) for n in self.lengths)
        self.pool = PagePool(max(pages, 1), page_size=page_size)
        self.stores = [KvStore(self.pool, hkv, head_dim, dtype=dtype, device=device) for _ in range(layers)]
        self.config = AttentionConfig(head_count=hq, head_dim=head_dim, page_size=page_size,
                                      kv_head_count=hkv)
        for local, n in enumerate(self.lengths):
            self.pool.reserve(local, n)
        self._batch = None

    @property
    def seq_ids(self) -> list:
        """Local sequence ids (0..len-1); global id = indices[local]."""
        return list(range(len(self.lengths)))

    def decode_batch(self):
        from .batch import DecodeBatch

        if self._batch is None:
            self._batch = DecodeBatch(self.stores, self.seq_ids, self.config)
        return self._batch

    def step(self, queries, k_new, v_new, **kw):
        """One decode step of this shard's sequences (K1 fused into K2 + K2c)."""
        return self.decode_batch().step(queries, k_new, v_new, **kw)

    def kv_report(self) -> dict:
        rep = kv_overhead([self.pool.table(s).logical_len or n for s, n in zip(self.seq_ids, self.lengths)],
                          self.pool.page_size)
        rep.update(rank=self.rank, sequences=len(self.indices))
        return rep


def gather_kv_reports(report: dict, group=None) -> dict:
    """All-gather per-shard KV reports; totals use the same definition."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        reports = [report]
    else:
        reports = [None] * dist.get_world_size(group)
        dist.all_gather_object(reports, report, group=group)
    tokens = sum(r["tokens"] for r in reports)
    charged = sum(r["charged_slots"] for r in reports)
    return {"shards": reports, "tokens": tokens, "charged_slots": charged,
            "overhead": (charged / tokens - 1.0) if tokens else 0.0}


def head_shard_range(hq: int, hkv: int, rank: int, world: int) -> tuple:
    """(q_head_lo, q_head_hi, kv_head_lo, kv_head_hi) owned by `rank` in
    head-sharded mode; kv heads split evenly, q heads follow (q head h reads
    kv head h // G)."""
    if hkv % world:
        raise ValueError(f"{hkv} kv heads do not split over {world} ranks")
    per = hkv // world
    g = hq // hkv
    return rank * per * g, (rank + 1) * per * g, rank * per, (rank + 1) * per


def head_shard_gather(out_local, group=None):
    """[B, hq/n, D] slice of every rank -> [B, hq, D] in head order.  NCCL
    all_gather_into_tensor over NVLink on GPUs; list all_gather elsewhere
    (gloo tests)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    x = out_local.contiguous()
    if x.is_cuda and dist.get_backend(group) == "nccl":
        buf = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(buf, x, group=group)
    else:
        parts = [torch.empty_like(x) for _ in range(world)]
        dist.all_gather(parts, x, group=group)
        buf = torch.stack(parts)
    # [n, B, h, D] -> [B, n*h, D]
    return buf.permute(1, 0, 2, 3).reshape(x.shape[0], world * x.shape[1], x.shape[2])


class HeadShard:
    """This rank's share of a head-sharded decode.

    Rank r owns kv heads [klo, khi) and the query heads that read them
    [qlo, qhi) of *every* sequence.  The allocator is replicated: every rank
    runs the same reserve/grow/append stream on its own pool, so block tables
    are identical everywhere and only the per-head K/V slices differ.  After
    the local decode the [B, hq/n, D] output slices are all-gathered over the
    process group (NCCL over NVLink on a B200 box)."""

    def __init__(self, lengths, *, rank: int, world: int, hq: int, hkv: int, head_dim: int, page_size: int,
                 dtype="bf16", device=None, headroom_tokens: int = 0):
        from .attention import AttentionConfig
        from .pool import PagePool
        from .store import KvStore

        self.rank, self.world = rank, world
        self.qlo, self.qhi, self.klo, self.khi = head_shard_range(hq, hkv, rank, world)
        self.lengths = [int(x) for x in lengths]
        pages = sum(-(-(n + headroom_tokens) // page_size) for n in self.lengths)
        self.pool = PagePool(max(pages, 1), page_size=page_size)
        self.store = KvStore(self.pool, self.khi - self.klo, head_dim, dtype=dtype, device=device)
        self.config = AttentionConfig(head_count=self.qhi - self.qlo, head_dim=head_dim, page_size=page_size,
                                      kv_head_count=self.khi - self.klo)
        for s, n in enumerate(self.lengths):
            self.pool.reserve(s, n)
        self._batch = None

    def assign(self, seq, positions, k_full, v_full) -> None:
        """Write this rank's head slice of full-width K/V rows [n, hkv, D]."""
        self.store.assign(seq, positions, k_full[:, self.klo:self.khi], v_full[:, self.klo:self.khi])

    def step_local(self, q_full, k_new_full, v_new_full, **kw):
        """Decode step of every sequence on this rank's heads -> [B, hq/n, D]."""
        from .batch import DecodeBatch

        if self._batch is None:
            self._batch = DecodeBatch(self.store, list(range(len(self.lengths))), self.config)
        return self._batch.step(q_full[:, self.qlo:self.qhi].contiguous(),
                                k_new_full[:, self.klo:self.khi].contiguous(),
                                v_new_full[:, self.klo:self.khi].contiguous(), **kw)

    def step(self, q_full, k_new_full, v_new_full, group=None, **kw):
        """Local decode + all-gather of the head slices -> [B, hq, D]."""
        import torch.distributed as dist

        out = self.step_local(q_full, k_new_full, v_new_full, **kw)
        if self.world > 1 and dist.is_available() and dist.is_initialized():
            return head_shard_gather(out, group)
        return out


def _event_seqs(ev):
    from .workload import ForkEvent

    return (ev.parent, ev.child) if isinstance(ev, ForkEvent) else (ev.seq,)


def shard_trace(trace, world: int) -> list:
    """Split a workload trace (its JSONL form is the sharder's wire format,
    reference workload.py:61-85) into `world` per-rank traces.

    Sequences linked by forks share pages, so each fork family stays on one
    rank; families are placed by LPT on the tokens they bring (prompts,
    decode bursts, fork prefixes).  Every rank keeps the events of its
    families in trace order, so its replay is exactly the global trace
    restricted to its sequences.  Deterministic: every rank computes the
    same split from the same document without communicating."""
    parent = {}

    def find(x):
        parent.setdefault(x, x)
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for ev in trace.events:
        seqs = _event_seqs(ev)
        roots = [find(s) for s in seqs]
        for r in roots[1:]:
            if r != roots[0]:
                parent[r] = roots[0]
    fams, weight = {}, []
    for ev in trace.events:
        f = find(_event_seqs(ev)[0])
        if f not in fams:
            fams[f] = len(weight)
            weight.append(0)
        n = getattr(ev, "prompt_len", None)
        n = getattr(ev, "n_tokens", n) if n is None else n
        n = getattr(ev, "prefix_len", n) if n is None else n
        weight[fams[f]] += int(n or 0)
    rank_of = [0] * len(weight)
    for r, part in enumerate(lpt_partition(weight, world)):
        for i in part:
            rank_of[i] = r
    out = [type(trace)(name=f"{trace.name}@{r}/{world}", seed=trace.seed, events=[]) for r in range(world)]
    for ev in trace.events:
        out[rank_of[fams[find(_event_seqs(ev)[0])]]].events.append(ev)
    return out
