"""Workload traces: the JSONL wire format, the seeded
generators and the memory audit against the reference's own outputs
(tests/golden/trace_cases.json, made by make_trace_golden.py from
pagedkv.workload, workload.py:55-404).  Host-only: runs on the native
allocator without a GPU."""

import json
import os

import pytest

from paper_2506_07311_b200 import InvalidTrace
from paper_2506_07311_b200 import workload as W

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "trace_cases.json")))
CFG = W.KvBytesConfig(**GOLDEN["bytes_config"])
CASES = GOLDEN["cases"]


def _ids():
    return [f"{c['generator'][0] if c['generator'] else 'fork'}-{i}" for i, c in enumerate(CASES)]


@pytest.mark.parametrize("case", CASES, ids=_ids())
def test_jsonl_round_trip_and_hash(case):
    t = W.Trace.from_jsonl(case["jsonl"])
    assert t.to_jsonl() == case["jsonl"]
    assert t.stable_hash() == case["hash"]
    assert t.total_tokens() == case["total_tokens"]


@pytest.mark.parametrize("case", [c for c in CASES if c["generator"]], ids=[i for i, c in zip(_ids(), CASES)
                                                                            if c["generator"]])
def test_generators_reproduce_reference_traces(case):
    name, args, kwargs = case["generator"]
    t = getattr(W, name)(*args, **kwargs)
    assert t.to_jsonl() == case["jsonl"]
    assert t.stable_hash() == case["hash"]


@pytest.mark.parametrize("case", CASES, ids=_ids())
@pytest.mark.parametrize("ps", ["1", "16", "64"])
def test_full_report_matches_reference(case, ps):
    t = W.Trace.from_jsonl(case["jsonl"])
    want = case["reports"][ps]
    got = W.full_report(t, int(ps), None, CFG).to_dict(include_series="series" in want["paged"])
    assert got == want


def test_invalid_documents_and_events():
    for doc in GOLDEN["invalid_documents"]:
        with pytest.raises(InvalidTrace):
            W.Trace.from_jsonl(doc)
    bad = W.Trace("bad", None, [W.Decode(seq="ghost", n_tokens=3)])
    with pytest.raises(InvalidTrace):
        W.account(bad, W.PagedModel(16), CFG)
    neg = W.Trace("neg", None, [W.Arrive(seq="a", prompt_len=-1)])
    with pytest.raises(InvalidTrace):
        W.account(neg, W.PagedModel(16), CFG)
    over = W.Trace("over", None, [W.Arrive(seq="a", prompt_len=10)])
    with pytest.raises(InvalidTrace):
        W.account(over, W.ContiguousModel(5), CFG)
    with pytest.raises(ValueError):
        W.account(over, W.ContiguousModel(0), CFG)
    with pytest.raises(ValueError):
        W.gen_mixed_batch(0, "zipf")
    with pytest.raises(ValueError):
        W.gen_chat_growth(10, 5)
