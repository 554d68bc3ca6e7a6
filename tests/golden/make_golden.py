"""Generate golden vectors by running the REAL reference (`pagedkv`).

Run in the build container, where the reference is mounted read-only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (committed, small):
  allocator_scripts.json  op streams + reference `PagePool.dump()` after each op
  store_scripts.npz       assign/fork/CoW scripts + final reference K/V arrays
  attention_cases.npz     reference `paged_attention`, `reference_attention`
                          and KernelStats on scattered instances (incl. the C1
                          decode shape, GQA folds and bf16-rounded inputs)

Nothing on the GPU box reads /root/reference: tests consume these files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = os.environ.get("PAGEDKV_REF", "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import pagedkv as R  # noqa: E402  (the reference itself)
from pagedkv import verify as RV  # noqa: E402

from oracle.attention import fold_gqa_queries, round_bf16, unfold_gqa_output  # noqa: E402
from oracle.workloads import scattered_instance  # noqa: E402


def _err_name(exc):
    return type(exc).__name__


# ---------------------------------------------------------------------------
# 1. allocator scripts
# ---------------------------------------------------------------------------

def _run_pool_op(pool, op):
    kind = op["op"]
    if kind == "reserve":
        return pool.reserve(op["seq"], op["len"])
    if kind == "grow":
        return pool.grow(op["seq"], op["len"])
    if kind == "free":
        return pool.free(op["seq"])
    if kind == "fork":
        return list(pool.fork(op["parent"], op["seq"], op["len"]).entries)
    if kind == "privatize":
        return pool.privatize(op["seq"], op["block"])
    if kind == "set_len":
        pool.table(op["seq"]).logical_len = op["len"]
        return None
    if kind == "translate":
        a = pool.translate(op["seq"], op["pos"])
        return [a.page_id, a.offset]
    raise ValueError(kind)


def _random_pool_ops(seed, n_ops, capacity, ps):
    rng = np.random.default_rng(seed)
    ops, live, nxt = [], [], 0
    for _ in range(n_ops):
        kind = str(rng.choice(["reserve", "grow", "free", "fork", "privatize", "set_len",
                               "translate", "reserve_dup", "free_ghost"]))
        if kind == "reserve" or not live:
            name = f"q{nxt}"; nxt += 1
            ops.append({"op": "reserve", "seq": name, "len": int(rng.integers(0, 7 * ps))})
            live.append(name)
        elif kind == "reserve_dup":
            ops.append({"op": "reserve", "seq": live[int(rng.integers(len(live)))], "len": 1})
        elif kind == "free_ghost":
            ops.append({"op": "free", "seq": "ghost"})
        elif kind == "grow":
            ops.append({"op": "grow", "seq": live[int(rng.integers(len(live)))],
                        "len": int(rng.integers(0, 10 * ps))})
        elif kind == "free":
            ops.append({"op": "free", "seq": live.pop(int(rng.integers(len(live))))})
        elif kind == "fork":
            name = f"q{nxt}"; nxt += 1
            ops.append({"op": "fork", "parent": live[int(rng.integers(len(live)))], "seq": name,
                        "len": int(rng.integers(-1, 6 * ps))})
            live.append(name)
        elif kind == "privatize":
            ops.append({"op": "privatize", "seq": live[int(rng.integers(len(live)))],
                        "block": int(rng.integers(0, 4))})
        elif kind == "set_len":
            ops.append({"op": "set_len", "seq": live[int(rng.integers(len(live)))],
                        "len": int(rng.integers(0, 6 * ps))})
        else:
            ops.append({"op": "translate", "seq": live[int(rng.integers(len(live)))],
                        "pos": int(rng.integers(-1, 6 * ps))})
    return ops


def _record_pool_script(name, capacity, ps, ops):
    pool = R.PagePool(capacity, page_size=ps)
    steps = []
    for op in ops:
        try:
            ret = _run_pool_op(pool, op)
            out = {"ok": True, "ret": ret}
        except (R.PagedKvError, ValueError, IndexError) as exc:
            out = {"ok": False, "err": _err_name(exc)}
        steps.append({"op": op, "out": out, "dump": pool.dump()})
    return {"name": name, "capacity": capacity, "page_size": ps, "steps": steps}


def allocator_scripts():
    scripts = []
    # failed grants reorder the free stack.
    a1 = [{"op": "reserve", "seq": "x", "len": 4 * 16},
          {"op": "reserve", "seq": "y", "len": 16},
          {"op": "free", "seq": "x"},
          {"op": "free", "seq": "y"},
          {"op": "reserve", "seq": "big", "len": 96},
          {"op": "reserve", "seq": "big2", "len": 96},
          {"op": "reserve", "seq": "big3", "len": 96},
          {"op": "reserve", "seq": "ok", "len": 16},
          {"op": "grow", "seq": "ok", "len": 200}]
    scripts.append(_record_pool_script("appendix_a1", 6, 16, a1))
    # fork / privatize / LIFO reuse
    fk = [{"op": "reserve", "seq": "p", "len": 12},
          {"op": "set_len", "seq": "p", "len": 12},
          {"op": "fork", "parent": "p", "seq": "c", "len": 6},
          {"op": "fork", "parent": "p", "seq": "d", "len": 8},
          {"op": "privatize", "seq": "c", "block": 0},
          {"op": "privatize", "seq": "d", "block": 1},
          {"op": "free", "seq": "p"},
          {"op": "fork", "parent": "ghost", "seq": "e", "len": 1},
          {"op": "fork", "parent": "c", "seq": "e", "len": 99},
          {"op": "fork", "parent": "c", "seq": "d", "len": 2},
          {"op": "fork", "parent": "c", "seq": "f", "len": -1},
          {"op": "reserve", "seq": "g", "len": 40},
          {"op": "translate", "seq": "g", "pos": 9},
          {"op": "translate", "seq": "g", "pos": 40}]
    scripts.append(_record_pool_script("fork_cow", 16, 4, fk))
    for seed, (cap, ps, n) in enumerate([(24, 4, 200), (64, 16, 250), (12, 8, 200),
                                         (200, 16, 250), (7, 4, 150)]):
        scripts.append(_record_pool_script(f"random{seed}", cap, ps,
                                           _random_pool_ops(100 + seed, n, cap, ps)))
    return scripts


# ---------------------------------------------------------------------------
# 2. store scripts (assign / fork / CoW / grow / free), K/V state
# ---------------------------------------------------------------------------

def store_script(seed, capacity=48, ps=4, h=2, d=3, n_ops=250):
    rng = np.random.default_rng(seed)
    pool = R.PagePool(capacity, page_size=ps)
    store = R.KvStore(pool, h, d)
    ops, arrays = [], {}
    live, nxt = [], 0
    for i in range(n_ops):
        kind = str(rng.choice(["reserve", "grow", "assign", "assign", "fork", "free"]))
        if kind == "reserve" or not live:
            op = {"op": "reserve", "seq": f"q{nxt}", "len": int(rng.integers(0, 5 * ps))}
            nxt += 1
        elif kind == "grow":
            s = live[int(rng.integers(len(live)))]
            op = {"op": "grow", "seq": s,
                  "len": len(pool.table(s).entries) * ps + int(rng.integers(0, 2 * ps))}
        elif kind == "assign":
            s = live[int(rng.integers(len(live)))]
            cap = len(pool.table(s).entries) * ps
            if cap == 0:
                continue
            cnt = int(rng.integers(1, min(cap, 3 * ps) + 1))
            pos = rng.integers(0, cap, cnt)  # duplicates allowed: last write wins
            op = {"op": "assign", "seq": s, "key": f"a{i}"}
            arrays[f"a{i}_pos"] = pos.astype(np.int64)
            arrays[f"a{i}_k"] = rng.standard_normal((cnt, h, d)).astype(np.float32)
            arrays[f"a{i}_v"] = rng.standard_normal((cnt, h, d)).astype(np.float32)
        elif kind == "fork":
            s = live[int(rng.integers(len(live)))]
            op = {"op": "fork", "parent": s, "seq": f"q{nxt}",
                  "len": int(rng.integers(0, pool.table(s).logical_len + 1))}
            nxt += 1
        else:
            op = {"op": "free", "seq": live.pop(int(rng.integers(len(live))))}
        try:
            if op["op"] == "reserve":
                pool.reserve(op["seq"], op["len"]); live.append(op["seq"])
            elif op["op"] == "grow":
                pool.grow(op["seq"], op["len"])
            elif op["op"] == "assign":
                k = op["key"]
                store.assign(op["seq"], arrays[k + "_pos"], arrays[k + "_k"], arrays[k + "_v"])
            elif op["op"] == "fork":
                pool.fork(op["parent"], op["seq"], op["len"]); live.append(op["seq"])
            else:
                pool.free(op["seq"])
            op["ok"] = True
        except R.PagedKvError as exc:
            op["ok"] = False
            op["err"] = _err_name(exc)
        ops.append(op)
    arrays["final_keys"] = store.keys.copy()
    arrays["final_values"] = store.values.copy()
    meta = {"capacity": capacity, "page_size": ps, "heads": h, "dim": d, "ops": ops,
            "final_dump": pool.dump(),
            "gathers": {s: pool.table(s).logical_len for s in live}}
    for s in live:
        gk, gv = store.gather(s, pool.table(s).logical_len)
        arrays[f"gather_{s}_k"] = gk
        arrays[f"gather_{s}_v"] = gv
    return meta, arrays


# ---------------------------------------------------------------------------
# 3. attention cases
# ---------------------------------------------------------------------------

ATTN_CASES = [
    # name, seed, lengths, hq, hkv, d, ps, causal, q_lengths, bf16
    ("c1_decode", 0, [512], 8, 8, 64, 16, True, [1], False),
    ("mixed_prefill_p16", 17, [37, 90, 5], 4, 4, 16, 16, True, None, False),
    ("mixed_prefill_p64_nc", 18, [120, 33], 4, 4, 16, 64, False, None, False),
    ("suffix_p128", 19, [299, 140, 12, 1], 4, 4, 16, 128, True, [7, 3, 12, 1], False),
    ("decode_batch_d64", 20, [300, 17, 64, 129], 8, 8, 64, 16, True, [1, 1, 1, 1], False),
    ("decode_batch_d8", 21, [40, 1, 33], 1, 1, 8, 16, True, [1, 1, 1], False),
    ("gqa_decode_bf16", 22, [200, 77, 513], 8, 2, 128, 16, True, [1, 1, 1], True),
    ("gqa_prefill_bf16", 23, [96, 40], 8, 2, 64, 16, True, None, True),
    ("mha_decode_bf16_d128", 24, [300, 129], 4, 4, 128, 16, True, [1, 1], True),
    ("noncausal_suffix_bf16", 25, [64, 50], 4, 1, 32, 16, False, [5, 50], True),
]


def attention_cases():
    arrays, index = {}, []
    for name, seed, lengths, hq, hkv, d, ps, causal, qlens, bf16 in ATTN_CASES:
        rng = np.random.default_rng(seed)
        inst = scattered_instance(
            rng, lengths, kv_heads=hkv, q_heads=hq, head_dim=d, page_size=ps, q_lengths=qlens,
            make_pool=lambda c, p: R.PagePool(c, page_size=p),
            make_store=lambda pool, h, dd: R.KvStore(pool, h, dd),
            cast=round_bf16 if bf16 else None)
        g = hq // hkv
        view = inst.store.batch_view(inst.seq_ids, inst.lengths)
        meta = R.MaskMeta.suffix(view, inst.q_lengths)
        cfg = R.AttentionConfig(head_count=hkv, head_dim=d, causal=causal, page_size=ps)
        stats = R.KernelStats()
        if g > 1:
            fmeta = R.MaskMeta(view=view, q_seq=np.repeat(meta.q_seq, g), q_pos=np.repeat(meta.q_pos, g))
            out = unfold_gqa_output(
                R.paged_attention(fold_gqa_queries(inst.queries, hkv), inst.store, fmeta, cfg,
                                  stats=stats), hq)
            kx = np.repeat(inst.keys, g, axis=1)
            vx = np.repeat(inst.values, g, axis=1)
        else:
            out = R.paged_attention(inst.queries, inst.store, meta, cfg, stats=stats)
            kx, vx = inst.keys, inst.values
        ref64 = R.reference_attention(inst.queries, kx, vx, inst.lengths, causal=causal,
                                      scale=cfg.scale, q_lengths=inst.q_lengths)
        # inputs are regenerated from the seed by the restated recipe; their
        # float64 checksums pin that regeneration
        arrays[f"{name}_out"] = out
        arrays[f"{name}_ref64"] = ref64
        index.append({
            "name": name, "seed": seed, "lengths": lengths, "q_lengths": inst.q_lengths,
            "hq": hq, "hkv": hkv, "d": d, "page_size": ps, "causal": causal, "bf16": bf16,
            "scale": cfg.scale, "pool_dump": inst.pool.dump(),
            "checksums": [float(np.sum(inst.queries, dtype=np.float64)),
                          float(np.sum(inst.keys, dtype=np.float64)),
                          float(np.sum(inst.values, dtype=np.float64))],
            "stats": {"visited_blocks": stats.visited_blocks, "skipped_blocks": stats.skipped_blocks,
                      "allowed_pairs": stats.allowed_pairs},
        })
    return index, arrays


def main():
    out = HERE
    scripts = allocator_scripts()
    with open(os.path.join(out, "allocator_scripts.json"), "w") as f:
        json.dump(scripts, f, separators=(",", ":"))
    metas, arrays = [], {}
    for seed in (1, 2, 3):
        meta, arr = store_script(seed)
        metas.append(meta)
        arrays.update({f"s{seed}_{k}": v for k, v in arr.items()})
    np.savez_compressed(os.path.join(out, "store_scripts.npz"), **arrays)
    with open(os.path.join(out, "store_scripts.json"), "w") as f:
        json.dump(metas, f, separators=(",", ":"))
    index, arrays = attention_cases()
    np.savez_compressed(os.path.join(out, "attention_cases.npz"), **arrays)
    with open(os.path.join(out, "attention_cases.json"), "w") as f:
        json.dump(index, f, separators=(",", ":"))
    # verify-harness scripts: the reference's own self-checks pass on this tree
    res = RV.run_allocator_script(seed=1, ops=500)
    assert res.ok, res
    print("golden vectors written to", out)


if __name__ == "__main__":
    main()
