"""Replay a workload trace on the device engine and audit it (SURVEY.md §8
f-3).  The trace is a reference-format JSONL document (`--trace`) or one of
the generators; `--gen c5` builds the C5 batch as a trace (512 prompts of
the C5 lengths, one decode token each, then finishes).  Reports the paged
account of the device pool next to the contiguous one (reference
full_report definitions) and the device time spent in K1 appends and
attention.

    python tools/trace_replay.py --gen c5 [--page-size 16] [--attend]
    python tools/trace_replay.py --trace t.jsonl
"""

import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_07311_b200 import workload as W  # noqa: E402
from paper_2506_07311_b200.workloads import config_lengths  # noqa: E402


def c5_trace():
    lens = config_lengths("c5")
    names = [f"s{i:03d}" for i in range(len(lens))]
    ev = [W.Arrive(s, n) for s, n in zip(names, lens)]
    ev += [W.Decode(s, 1) for s in names]
    ev += [W.Finish(s) for s in names]
    return W.Trace("c5_batch", 0, ev)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trace")
    ap.add_argument("--gen", default="c5", choices=["c5", "ladder", "uniform", "chat"])
    ap.add_argument("--page-size", type=int, default=16)
    ap.add_argument("--attend", action="store_true")
    ap.add_argument("--out")
    a = ap.parse_args()
    if a.trace:
        trace = W.Trace.from_jsonl(open(a.trace).read())
    else:
        trace = {"c5": c5_trace, "ladder": lambda: W.gen_mixed_batch(0, "ladder"),
                 "uniform": lambda: W.gen_mixed_batch(0, "uniform"),
                 "chat": lambda: W.gen_chat_growth(128, 32768)}[a.gen]()
    hq, hkv, d = 32, 8, 128
    cfg = W.KvBytesConfig(layers=1, head_count=hkv, head_dim=d, bytes_per_scalar=2)
    rep = W.DeviceReplay(trace, page_size=a.page_size, hq=hq, hkv=hkv, head_dim=d, dtype="bf16",
                         attend=a.attend)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    paged = rep.run(cfg)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    report = W.full_report(trace, a.page_size, None, cfg, paged=paged)
    out = {
        "trace": trace.name, "trace_hash": trace.stable_hash(), "events": len(trace.events),
        "page_size": a.page_size, "layout": f"GQA {hq}q/{hkv}kv x{d} bf16, one layer",
        "paged": report.paged.to_dict(False), "contiguous": report.contiguous.to_dict(False),
        "device_ms": round(e0.elapsed_time(e1), 2), "wall_s": round(wall, 2), **rep.stats,
        "append_GBps_device": round(rep.stats["appended_tokens"] * hkv * d * 2 * 2 / (e0.elapsed_time(e1) * 1e6), 1),
    }
    print(json.dumps(out))
    if a.out:
        with open(a.out, "w") as f:
            f.write(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
