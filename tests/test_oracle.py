"""Pin the CPU oracle (oracle/) to the real reference: golden vectors always,
the live reference when it is mounted (build container only)."""

import os

import numpy as np
import pytest

from oracle import OracleMeta, OraclePool, OracleStore, dense_attention_f64, relative_error
from oracle.attention import (
    fold_gqa_meta,
    fold_gqa_queries,
    round_bf16,
    streaming_attention,
    unfold_gqa_output,
)
from oracle.workloads import config_lengths, lpt_partition, scattered_instance

from replay import replay_pool_script, replay_store_script

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _oracle_pool(c, p):
    return OraclePool(c, p)


def _oracle_store(pool, h, d):
    return OracleStore(pool, h, d)


def test_oracle_allocator_matches_golden(golden_allocator):
    n = 0
    for script in golden_allocator:
        for step, out, dump in replay_pool_script(script, _oracle_pool):
            assert out == step["out"], (script["name"], step["op"])
            assert dump == step["dump"], (script["name"], step["op"])
            n += 1
    assert n > 1000


def test_oracle_store_matches_golden(golden_store):
    metas, arrays = golden_store
    for i, meta in enumerate(metas):
        pre = f"s{i + 1}_"
        pool, store = replay_store_script(meta, arrays, pre, _oracle_pool, _oracle_store)
        assert pool.dump() == meta["final_dump"]
        assert np.array_equal(store.keys, arrays[pre + "final_keys"])
        assert np.array_equal(store.values, arrays[pre + "final_values"])
        for seq, length in meta["gathers"].items():
            gk, gv = store.gather(seq, length)
            assert np.array_equal(gk, arrays[f"{pre}gather_{seq}_k"])
            assert np.array_equal(gv, arrays[f"{pre}gather_{seq}_v"])


def build_oracle_case(case):
    rng = np.random.default_rng(case["seed"])
    inst = scattered_instance(
        rng, case["lengths"], kv_heads=case["hkv"], q_heads=case["hq"], head_dim=case["d"],
        page_size=case["page_size"], q_lengths=case["q_lengths"], make_pool=_oracle_pool,
        make_store=_oracle_store, cast=round_bf16 if case["bf16"] else None)
    return inst


def test_oracle_attention_matches_golden(golden_attention):
    index, arrays = golden_attention
    for case in index:
        inst = build_oracle_case(case)
        # the restated scatter recipe reproduces the reference's tables and inputs
        assert inst.pool.dump() == case["pool_dump"], case["name"]
        sums = [float(np.sum(a, dtype=np.float64)) for a in (inst.queries, inst.keys, inst.values)]
        assert sums == case["checksums"], case["name"]
        view = inst.store.batch_view(inst.seq_ids, inst.lengths)
        meta = OracleMeta.suffix(view, inst.q_lengths)
        g = case["hq"] // case["hkv"]
        rows = inst.store.view_row_indices(view)
        stats = {}
        out = unfold_gqa_output(streaming_attention(
            fold_gqa_queries(inst.queries, case["hkv"]), inst.store.keys[rows],
            inst.store.values[rows], fold_gqa_meta(meta, g), scale=case["scale"],
            causal=case["causal"], tile=case["page_size"], stats=stats), case["hq"])
        ref_out = arrays[case["name"] + "_out"]
        # same algorithm, same BLAS: expect bit-equality, tolerate BLAS drift
        assert relative_error(out, ref_out) <= 1e-6, case["name"]
        assert stats == case["stats"], case["name"]
        ref64 = dense_attention_f64(inst.queries, inst.keys, inst.values, inst.lengths,
                                    causal=case["causal"], scale=case["scale"],
                                    q_lengths=inst.q_lengths)
        assert relative_error(ref64, arrays[case["name"] + "_ref64"]) <= 1e-12, case["name"]
        assert relative_error(out, ref64) <= 1e-5, case["name"]


def test_config_lengths_match_survey():
    c2 = config_lengths("c2")
    assert len(c2) == 32 and sum(c2) == 36477
    c5 = config_lengths("c5")
    assert len(c5) == 512 and sum(c5) == 3431895


def test_lpt_partition_balance():
    c5 = config_lengths("c5")
    for n in (2, 4, 8):
        parts = lpt_partition(c5, n)
        assert sorted(i for p in parts for i in p) == list(range(512))
        loads = [sum(c5[i] for i in p) for p in parts]
        assert max(loads) / (sum(loads) / n) < 1.001


def test_round_bf16_matches_torch():
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(0).standard_normal(4096).astype(np.float32) * 100
    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(round_bf16(x), want)


# ---- live reference (build container only) ---------------------------------

def test_oracle_vs_live_reference_random_instances(live_reference):
    R = live_reference
    from pagedkv.verify import build_attention_instance, relative_error as ref_rel

    for seed in range(6):
        rng = np.random.default_rng(1000 + seed)
        lengths = [int(x) for x in rng.integers(1, 200, 3)]
        causal = bool(seed % 2)
        inst = build_attention_instance(np.random.default_rng(seed), lengths, head_count=2,
                                        head_dim=8, page_size=16, causal=causal)
        want = inst.paged_output()
        oinst = scattered_instance(np.random.default_rng(seed), lengths, kv_heads=2, head_dim=8,
                                   page_size=16, make_pool=_oracle_pool, make_store=_oracle_store)
        assert oinst.pool.dump() == inst.pool.dump()
        view = oinst.store.batch_view(oinst.seq_ids, oinst.lengths)
        meta = OracleMeta.suffix(view, oinst.q_lengths)
        rows = oinst.store.view_row_indices(view)
        got = streaming_attention(oinst.queries, oinst.store.keys[rows], oinst.store.values[rows],
                                  meta, scale=inst.config.scale, causal=causal, tile=16)
        assert np.array_equal(got, want)
        assert ref_rel(got, inst.reference_output()) <= 1e-5


def test_oracle_allocator_vs_live_reference_script(live_reference):
    """A fresh random op stream (not in the golden set), replayed on the real
    reference and on the oracle; dumps must agree after every op."""
    R = live_reference
    rng = np.random.default_rng(77)
    ops, live = [], []
    for i in range(800):
        kind = str(rng.choice(["reserve", "grow", "free", "fork", "privatize", "set_len"]))
        if kind == "reserve" or not live:
            ops.append({"op": "reserve", "seq": f"s{i}", "len": int(rng.integers(0, 60))})
            live.append(f"s{i}")
        elif kind == "grow":
            ops.append({"op": "grow", "seq": live[int(rng.integers(len(live)))],
                        "len": int(rng.integers(0, 90))})
        elif kind == "free":
            ops.append({"op": "free", "seq": live.pop(int(rng.integers(len(live))))})
        elif kind == "fork":
            ops.append({"op": "fork", "parent": live[int(rng.integers(len(live)))],
                        "seq": f"s{i}", "len": int(rng.integers(0, 40))})
            live.append(f"s{i}")
        elif kind == "privatize":
            ops.append({"op": "privatize", "seq": live[int(rng.integers(len(live)))],
                        "block": int(rng.integers(0, 3))})
        else:
            ops.append({"op": "set_len", "seq": live[int(rng.integers(len(live)))],
                        "len": int(rng.integers(0, 40))})
    from replay import run_pool_op

    a, b = R.PagePool(40, page_size=8), OraclePool(40, 8)
    for op in ops:
        outs = []
        for pool in (a, b):
            try:
                outs.append(("ok", run_pool_op(pool, op)))
            except Exception as exc:
                outs.append(("err", type(exc).__name__))
        assert outs[0] == outs[1], op
        assert a.dump() == b.dump(), op


def test_product_workloads_and_sharder_match_oracle():
    """The product-side generator / LPT sharder agree with the oracle's copies."""
    from oracle.workloads import config_lengths as o_lengths, lpt_partition as o_lpt
    from paper_2506_07311_b200.sharding import lpt_partition, shard_balance
    from paper_2506_07311_b200.workloads import config_lengths as p_lengths

    for name in ("c1", "c2", "c5"):
        assert p_lengths(name) == o_lengths(name)
    c5 = p_lengths("c5")
    for n in (1, 2, 4, 8):
        assert lpt_partition(c5, n) == o_lpt(c5, n)
        assert shard_balance(c5, lpt_partition(c5, n)) < 1.001


def test_toy_decoder_restatement_matches_reference_golden():
    """The test-side toy model (tests/toy_decoder.py) reproduces the real
    reference's no-cache logits, so it can drive DecodeSession on the GPU."""
    from toy_decoder import ToyDecoder, load_cases

    for case in load_cases(os.path.join(GOLDEN_DIR, "decoder_cases.npz")):
        dec = ToyDecoder(case["config"])
        toks = [int(t) for t in case["tokens"]]
        for i, want in enumerate(case["nocache"]):
            got = dec.forward_nocache(toks[: case["n_prompt"] + 10 * i])
            assert relative_error(got, want) <= 1e-5, case["name"]
        # greedy decode of the golden cached run is self-consistent
        assert all(int(np.argmax(case["logits"][i])) == toks[case["n_prompt"] + i]
                   for i in range(case["steps"]))


def test_package_reference_attention_matches_golden_float64(golden_attention):
    """The package's dense float64 diagnostic (reference attention.py:389-447)
    reproduces the real reference's reference_attention outputs."""
    from paper_2506_07311_b200 import reference_attention

    index, arrays = golden_attention
    for case in index:
        inst = build_oracle_case(case)
        got = reference_attention(inst.queries, inst.keys, inst.values, inst.lengths, causal=case["causal"],
                                  scale=case["scale"], q_lengths=inst.q_lengths, device="cpu")
        assert relative_error(got.numpy(), arrays[case["name"] + "_ref64"]) <= 1e-12, case["name"]
