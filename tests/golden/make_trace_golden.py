"""Golden workload traces and memory accounts from the REAL reference
(`pagedkv.workload`).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_trace_golden.py

Writes trace_cases.json: for each generated trace its JSONL text, the
reference `Trace.stable_hash()` (workload.py:84-85) and the reference
`full_report(...).to_dict()` (workload.py:379-404) at several page sizes,
plus one hand-written trace with forks.  Tests check the engine's trace
codec, generators and its device-pool replay against these numbers.
"""

from __future__ import annotations

import json
import os
import sys

REF = os.environ.get("PAGEDKV_REF", "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from pagedkv import workload as W  # noqa: E402  (the reference itself)


def fork_trace():
    t = W.Trace(name="fork_family", seed=7)
    ev = t.events
    ev.append(W.Arrive(seq="root", prompt_len=1000))
    ev.append(W.ForkEvent(parent="root", child="a", prefix_len=1000))
    ev.append(W.ForkEvent(parent="root", child="b", prefix_len=515))
    ev.append(W.Decode(seq="a", n_tokens=77))
    ev.append(W.Decode(seq="b", n_tokens=300))
    ev.append(W.Arrive(seq="solo", prompt_len=33))
    ev.append(W.Finish(seq="root"))
    ev.append(W.ForkEvent(parent="a", child="c", prefix_len=1077))
    ev.append(W.Decode(seq="c", n_tokens=5))
    ev.append(W.Finish(seq="a"))
    ev.append(W.Finish(seq="solo"))
    ev.append(W.Finish(seq="b"))
    ev.append(W.Finish(seq="c"))
    return t


def main():
    traces = [
        W.gen_single_sequence(4097),
        W.gen_single_sequence(0, seq_id="empty"),
        W.gen_mixed_batch(0, "ladder"),
        W.gen_mixed_batch(3, "ladder"),
        W.gen_mixed_batch(0, "uniform"),
        W.gen_mixed_batch(11, "uniform", count=24),
        W.gen_chat_growth(100, 9000),
        W.gen_chat_growth(7, 1000, step_factor=1.7, seq_id="c2"),
        fork_trace(),
    ]
    gens = [
        ["gen_single_sequence", [4097], {}],
        ["gen_single_sequence", [0], {"seq_id": "empty"}],
        ["gen_mixed_batch", [0, "ladder"], {}],
        ["gen_mixed_batch", [3, "ladder"], {}],
        ["gen_mixed_batch", [0, "uniform"], {}],
        ["gen_mixed_batch", [11, "uniform"], {"count": 24}],
        ["gen_chat_growth", [100, 9000], {}],
        ["gen_chat_growth", [7, 1000], {"step_factor": 1.7, "seq_id": "c2"}],
        None,
    ]
    cfg = W.KvBytesConfig(layers=32, head_count=8, head_dim=128, bytes_per_scalar=2)
    cases = []
    for t, g in zip(traces, gens):
        reports = {}
        for ps in (1, 16, 64):
            rep = W.full_report(t, ps, None, cfg).to_dict(include_series=len(t.events) <= 40)
            reports[str(ps)] = rep
        cases.append({"generator": g, "jsonl": t.to_jsonl(), "hash": t.stable_hash(),
                      "total_tokens": t.total_tokens(), "reports": reports})
    bad = [
        '{"seed": 0, "trace": "x"}\n{"event": "teleport", "seq": "a"}\n',
        "",
    ]
    out = {"bytes_config": {"layers": 32, "head_count": 8, "head_dim": 128, "bytes_per_scalar": 2},
           "cases": cases, "invalid_documents": bad}
    with open(os.path.join(HERE, "trace_cases.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("wrote", len(cases), "traces")


if __name__ == "__main__":
    main()
