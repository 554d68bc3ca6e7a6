"""Host planner of the tensor-core decode (no GPU): the stream-K style
segment partition covers every (query, head item) page exactly once, pieces
of a cut unit get consecutive partial slots and one combine record, and CTA
loads are balanced."""

import numpy as np
import pytest

from paper_2506_07311_b200 import _lib
from paper_2506_07311_b200.workloads import config_lengths

HDR = 14


def parse(plan):
    hb, wph, qgs, qgroups, head_items, total, ncomb, nq, grid, cta_off, items_off, comb_off, ctr_off, cluster = plan[:HDR]
    nk = plan[HDR:HDR + nq]
    cta = plan[cta_off:cta_off + grid + 1]
    items = plan[items_off:items_off + 6 * total].reshape(-1, 6)
    assert (plan[ctr_off:ctr_off + 8 * ncomb] == 0).all() and ctr_off + 8 * ncomb == plan.size
    comb = plan[comb_off:comb_off + 4 * ncomb].reshape(-1, 4)
    return dict(hb=hb, wph=wph, head_items=head_items, nq=nq, grid=grid, nk=nk, cta=cta, items=items, comb=comb,
                cluster=cluster)


CASES = [
    ("c2", config_lengths("c2"), 32, 32),
    ("c3-b64", [8192] * 64, 32, 8),
    ("c3-b1-32k", [32768], 32, 8),
    ("c5", config_lengths("c5"), 32, 8),
    ("tiny", [1, 2, 17], 8, 2),
    ("many", list(np.random.default_rng(3).integers(1, 40, 2500)), 4, 2),
]


@pytest.mark.parametrize("name,lengths,hq,hkv", CASES, ids=[c[0] for c in CASES])
def test_segment_plan_covers_every_page_once(name, lengths, hq, hkv):
    check_plan(lengths, hq, hkv, 16, balance=True)


@pytest.mark.timeout(300, method="thread")  # a planner that never terminates must fail, not hang
def test_planner_fuzz_terminates_and_covers():
    """Random batches, page sizes and head shapes.  Regression: a CTA
    capacity below per-item overhead + minimum piece used to open empty
    CTAs forever (75 x 75-key queries, 8 heads, D 8, page 16 hung)."""
    rng = np.random.default_rng(11)
    check_plan([75] * 75, 8, 8, 16)
    for _ in range(300):
        nq = int(rng.integers(1, 300))
        lengths = np.maximum(1, np.exp(rng.uniform(0, np.log(40000), nq))).astype(np.int32)
        if rng.random() < 0.3:
            lengths[:] = lengths[0]
        ps = int(rng.choice([8, 16, 32, 64, 128]))
        hq, hkv = [(8, 8), (32, 8), (32, 32), (16, 2), (4, 1), (48, 2)][int(rng.integers(6))]
        check_plan(lengths, hq, hkv, ps)


@pytest.mark.parametrize("name,lengths,hq,hkv", CASES, ids=[c[0] for c in CASES])
def test_head_dim_64_plans_cover_and_use_the_smaller_page_cost(name, lengths, hq, hkv):
    """The planner's byte costs follow the head dim: a D = 64 page streams
    half the bytes, so the fixed per-item cost is twice as many pages and a
    D = 64 plan cuts units no more often than the D = 128 plan."""
    p64 = check_plan(lengths, hq, hkv, 16, head_dim=64)
    p128 = parse(_lib.attention_plan(np.asarray(lengths, np.int32), np.arange(len(lengths), dtype=np.int32), 16,
                                     hq, hkv, head_dim=128))
    assert len(p64["comb"]) <= len(p128["comb"])


def check_plan(lengths, hq, hkv, ps, balance=False, head_dim=128):
    nk = np.asarray(lengths, dtype=np.int32)
    plan = _lib.attention_plan(nk, np.arange(nk.size, dtype=np.int32), ps, hq, hkv, head_dim=head_dim)
    P = parse(plan)
    assert P["nq"] == nk.size and np.array_equal(P["nk"], nk)
    items, comb = P["items"], P["comb"]
    cta = P["cta"]
    assert cta[0] == 0 and cta[-1] == len(items) and (np.diff(cta) >= 0).all()
    pages = -(-nk.astype(np.int64) // ps)
    covered = {}
    for q, h, p0, p1, slot, ci in items:
        assert 0 <= p0 <= p1 <= pages[q] and (p0 < p1 or P["cluster"] > 1)
        covered.setdefault((q, h), []).append((p0, p1, slot))
        assert (slot < 0) == (ci < 0) and (ci < 0 or tuple(comb[ci][:2]) == (q, h))
    assert len(covered) == nk.size * P["head_items"]
    comb_map = {(q, h): (s0, n) for q, h, s0, n in comb}
    slots = []
    for (q, h), pieces in covered.items():
        assert pieces[0][0] == 0 and pieces[-1][1] == pages[q]
        assert all(a[1] == b[0] for a, b in zip(pieces, pieces[1:]))  # contiguous, in order
        if P["cluster"] > 1:  # one cluster of CTAs per unit, merged through DSMEM
            assert len(pieces) == P["cluster"] and all(p[2] == -1 for p in pieces)
        elif len(pieces) == 1:
            assert pieces[0][2] == -1 and (q, h) not in comb_map
        else:
            s0, n = comb_map[(q, h)]
            assert n == len(pieces) and [p[2] for p in pieces] == list(range(s0, s0 + n))
            slots += list(range(s0, s0 + n))
    assert sorted(slots) == list(range(len(slots)))
    # balance: bytes per CTA within one max piece of the mean
    load = np.zeros(P["grid"])
    for c in range(P["grid"]):
        for q, h, p0, p1, _, _ in items[cta[c]:cta[c + 1]]:
            load[c] += p1 - p0
    if balance and P["grid"] > 1 and P["cluster"] == 1:
        assert load.max() <= load.mean() * 1.15 + 64, (load.max(), load.mean())
    if P["cluster"] > 1:
        assert P["grid"] == len(items) <= 148 and P["grid"] % P["cluster"] == 0
    # few items per CTA
    assert len(items) <= nk.size * P["head_items"] + 2 * P["grid"]
    return P


@pytest.mark.parametrize("L,B", [(2048, 64), (4096, 32), (16384, 16), (8192, 64)])
def test_whole_units_for_uniform_batches_near_the_sm_count(L, B):
    """~128 equal (query, head block) units on 148 SMs: one uncut unit per
    CTA (no partials, no merges) — HBM saturates with ~120 CTAs, so cutting
    units to reach the last SMs only adds merges."""
    plan = _lib.attention_plan(np.full(B, L, np.int32), np.arange(B, dtype=np.int32), 16, 32, 8, 0)
    P = parse(plan)
    units = B * P["head_items"]
    assert P["grid"] == units == len(P["items"]) and len(P["comb"]) == 0
    assert (np.diff(P["cta"]) == 1).all()
    check_plan([L] * B, 32, 8, 16)


def test_mixed_lengths_keep_the_segment_schedule():
    """C2 (32 mixed lengths): unit sizes differ, so units are still cut to
    balance bytes across every SM."""
    plan = _lib.attention_plan(np.asarray(config_lengths("c2"), np.int32), np.arange(32, dtype=np.int32),
                               16, 32, 32, 0)
    P = parse(plan)
    assert P["grid"] == 148 and len(P["comb"]) > 0
