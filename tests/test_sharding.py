"""Request sharder and head-sharded gather (SURVEY.md §8 e) on CPU: a
world_size-2 gloo process group stands in for the NCCL group of the box."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2506_07311_b200.sharding import (  # noqa: E402
    gather_kv_reports,
    head_shard_gather,
    head_shard_range,
    kv_overhead,
    lpt_partition,
    shard_balance,
)
from paper_2506_07311_b200.workloads import config_lengths  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lens = config_lengths("c5")
        mine = lpt_partition(lens, world)[rank]
        # every rank derives the same partition without communication
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        # per-shard KV report, totals with the reference definition
        rep = kv_overhead([lens[i] for i in mine], 16)
        rep["rank"] = rank
        total = gather_kv_reports(rep)
        # head-sharded output gather: rank r owns q heads [lo, hi)
        B, hq, hkv, d = 3, 8, 4, 5
        lo, hi, klo, khi = head_shard_range(hq, hkv, rank, world)
        full = torch.arange(B * hq * d, dtype=torch.float32).reshape(B, hq, d)
        got = head_shard_gather(full[:, lo:hi].clone())
        q.put((rank, parts, total, bool(torch.equal(got, full)), (lo, hi, klo, khi)))
    finally:
        dist.destroy_process_group()


def test_two_rank_request_sharding_and_head_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lens = config_lengths("c5")
    for rank, parts, total, gathered_ok, rng in results:
        assert parts == lpt_partition(lens, world)
        flat = sorted(i for part in parts for i in part)
        assert flat == list(range(len(lens)))  # disjoint cover
        assert total["tokens"] == sum(lens) == 3431895
        assert abs(total["overhead"] - kv_overhead(lens, 16)["overhead"]) < 1e-12
        assert total["overhead"] < 0.05  # < 5% over the theoretical minimum
        assert gathered_ok
    assert sorted(r[4] for r in results) == [(0, 4, 0, 2), (4, 8, 2, 4)]


def test_lpt_balance_and_overhead_numbers():
    lens = config_lengths("c5")
    for n in (2, 4, 8):
        assert shard_balance(lens, lpt_partition(lens, n)) < 1.001
    rep = kv_overhead(lens, 16)
    assert rep["charged_slots"] == 214731 * 16
    assert abs(rep["overhead"] - 0.00111) < 5e-5
    with pytest.raises(ValueError):
        head_shard_range(32, 8, 0, 3)
    assert lpt_partition([5, 5, 5], 2) == [[0, 2], [1]]


def _trace_worker(rank, world, port, q):
    from paper_2506_07311_b200 import workload as W
    from paper_2506_07311_b200.sharding import shard_trace

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank 0 owns the trace; the JSONL document is the wire format
        doc = [None]
        if rank == 0:
            t = W.gen_mixed_batch(11, "uniform", count=24)
            fam = W.Trace("f", None, [W.Arrive("root", 1000), W.ForkEvent("root", "a", 1000),
                                      W.ForkEvent("a", "b", 515), W.Decode("b", 40), W.Finish("root"),
                                      W.Finish("a"), W.Finish("b")])
            t.events = fam.events[:3] + t.events + fam.events[3:]
            doc = [t.to_jsonl()]
        dist.broadcast_object_list(doc, src=0)
        trace = W.Trace.from_jsonl(doc[0])
        mine = shard_trace(trace, world)[rank]
        acct = W.account(mine, W.PagedModel(16), W.KvBytesConfig())  # replays cleanly on its own
        seqs = sorted({s for ev in mine.events for s in
                       ((ev.parent, ev.child) if isinstance(ev, W.ForkEvent) else (ev.seq,))})
        rep = {"tokens": mine.total_tokens(), "seqs": seqs, "peak": acct.peak_live_tokens,
               "events": len(mine.events), "hash": trace.stable_hash()}
        reps = [None] * world
        dist.all_gather_object(reps, rep)
        q.put((rank, reps, trace.total_tokens(), len(trace.events)))
    finally:
        dist.destroy_process_group()


def test_two_rank_trace_sharding_over_the_jsonl_wire():
    """A trace is broadcast as JSONL, every rank derives the same shard
    split (fork families kept whole), replays and audits its shard alone."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_trace_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, reps, total, n_events in results:
        assert len({r["hash"] for r in reps}) == 1
        assert sum(r["tokens"] for r in reps) == total
        assert sum(r["events"] for r in reps) == n_events
        s0, s1 = set(reps[0]["seqs"]), set(reps[1]["seqs"])
        assert not (s0 & s1) and len(s0 | s1) == 24 + 3
        assert {"root", "a", "b"} <= s0 or {"root", "a", "b"} <= s1  # the fork family stays together
        assert min(r["tokens"] for r in reps) > 0.3 * total  # LPT balance
