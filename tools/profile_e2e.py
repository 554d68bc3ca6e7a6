"""Host-side profile of the e2e decode step (DecodeBatch.step on C2) — where
the wall-clock time of one public-API step goes beyond the device time."""

import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    from paper_2506_07311_b200.batch import DecodeBatch
    from paper_2506_07311_b200.workloads import CONFIG_SHAPES, config_lengths

    lengths = config_lengths("c2")
    hq, hkv, d, ps, _ = CONFIG_SHAPES["c2"]
    pool, store, cfg = bench.build_cache(lengths, hq, hkv, d, ps, extra_tokens=80, device=dev)
    B = len(lengths)
    batch = DecodeBatch(store, list(range(B)), cfg)
    rng = np.random.default_rng(7)
    q = torch.from_numpy(rng.standard_normal((B, hq, d)).astype(np.float32)).bfloat16().pin_memory()
    k = torch.from_numpy(rng.standard_normal((B, hkv, d)).astype(np.float32)).bfloat16().pin_memory()
    out_host = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()

    def step():
        qd = q.to(dev, non_blocking=True)
        kd = k.to(dev, non_blocking=True)
        vd = k.to(dev, non_blocking=True)
        o = batch.step(qd, kd, vd)
        out_host.copy_(o, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()

    for _ in range(5):
        step()
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    print("wall us per step: median %.1f min %.1f" % (1e6 * np.median(ts), 1e6 * min(ts)))
    # host-only cost: launch without waiting
    t0 = time.perf_counter()
    for _ in range(30):
        qd = q.to(dev, non_blocking=True)
        o = batch.step(qd, k.to(dev, non_blocking=True), k.to(dev, non_blocking=True))
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print("host-only us per step (async): %.1f" % (1e6 * (t1 - t0) / 30))
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(30):
        step()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
