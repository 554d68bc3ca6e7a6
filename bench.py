"""Benchmark of the paged-attention hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c5] [--context L] [--batch B] [--sweep]

Workload (default, BASELINE.json configs[1] = C2): LLaMA-7B-shaped decode
attention, 32 heads x 128, bf16 KV cache, batch 32 with mixed contexts
128-2048 (seed-0 draw, sum 36,477 tokens), page size 16, scattered pages.  One
step = append one new token per sequence (K1) + split-K paged decode over the
whole context (plan + K2 + K2c), i.e. one decode step of one attention layer.

* `value`   whole-job KV-read GB/s with inputs resident in HBM (device-timed
            with CUDA events per step; L2 flushed between steps);
* `e2e`     the same metric through the public API (`DecodeBatch.step`) with
            pinned host inputs, H2D + D2H inside the timed region;
* `roofline` the dominant kernel (K2 decode) against the measured HBM copy
            bandwidth in MEASURED_PEAKS.json;
* `cpu_baseline` the oracle port of the reference CPU kernel on the host.

Multi-GPU: one process per GPU (torchrun); every rank runs its own C2 batch
(request sharding, no data-path collective), scaling "weak"; time = max over
ranks.  `--config c5` runs the 512-sequence request-sharded config instead
(LPT shards, strong scaling).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attn KV-read GB/s (% of 8 TB/s) and tokens/sec vs context 128-32k, 1/2/4/8 GPU"
NOMINAL_HBM_GBS = 8000.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c5"])
    ap.add_argument("--context", type=int, default=8192, help="c3 context length")
    ap.add_argument("--batch", type=int, default=16, help="c3 batch")
    ap.add_argument("--sweep", action="store_true", help="also print a C3 context sweep (stderr)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-prefill", action="store_true", help="skip the C4 prefill (K3) side measurement")
    ap.add_argument("--waves", type=int, default=0, help="split planner target waves (0 = default)")
    ap.add_argument("--heads", default="", help="experiment: override query:kv heads, e.g. 32:32")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def workload(args, rank: int, world: int):
    from paper_2506_07311_b200.sharding import lpt_partition
    from paper_2506_07311_b200.workloads import CONFIG_SHAPES, config_lengths

    if args.config == "c3":
        lengths = config_lengths("c3", batch=args.batch, context=args.context)
        name = f"C3 Llama-3-8B GQA 32q/8kv x128 bf16 decode, batch {args.batch}, context {args.context}, page 16"
    elif args.config == "c5":
        all_lens = config_lengths("c5")
        parts = lpt_partition(all_lens, world)
        lengths = [all_lens[i] for i in parts[rank]]
        name = "C5 request-sharded decode, 512 sequences, contexts 128-32k (LPT shards), GQA 32q/8kv x128 bf16, page 16"
    else:
        lengths = config_lengths("c2")
        name = "C2 LLaMA-7B MHA 32x128 bf16 decode, batch 32, mixed contexts 128-2048 (seed 0), page 16"
    hq, hkv, d, ps, _ = CONFIG_SHAPES[args.config]
    if args.heads:  # experiment override "HQ:HKV" (not a BASELINE config)
        hq, hkv = (int(x) for x in args.heads.split(":"))
        name += f" [heads overridden to {hq}q/{hkv}kv]"
    return name, lengths, hq, hkv, d, ps


def algorithmic_bytes(lengths, hq, hkv, d, ps, s=2, out_bytes=4):
    """KV + Q + O + block-table + length bytes of one step."""
    B = len(lengths)
    kv = sum(2 * n * hkv * d * s for n in lengths)
    return kv + B * hq * d * s + B * hq * d * out_bytes + 4 * sum(-(-n // ps) for n in lengths) + 4 * B, kv


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ---------------------------------------------------------------------------

class ClockSampler:
    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000010: "sync_boost", 0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown", 0x0000000000000080: "hw_power_brake_slowdown",
        0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.0005)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------

def build_cache(lengths, hq, hkv, d, ps, extra_tokens, device, seed=0):
    """Scattered pool + bf16 store holding `lengths` tokens per sequence."""
    import torch

    from paper_2506_07311_b200 import AttentionConfig, KvStore, PagePool

    B = len(lengths)
    need = sum(-(-(n + extra_tokens) // ps) for n in lengths)
    pad = max(B, need // 8)
    pool = PagePool(need + pad + 8, page_size=ps)
    store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=device)
    gen = torch.Generator(device=device).manual_seed(seed)
    # interleave throw-away reservations so tables point at scattered pages
    for b, n in enumerate(lengths):
        pool.reserve(("pad", b), ps * (1 + (b * 7919) % max(1, pad // B)))
        pool.reserve(b, n)
    for b in range(B):
        pool.free(("pad", b))
    chunk = 1 << 15
    for b, n in enumerate(lengths):
        for s0 in range(0, n, chunk):
            m = min(chunk, n - s0)
            k = torch.randn((m, hkv, d), generator=gen, device=device, dtype=torch.bfloat16)
            v = torch.randn((m, hkv, d), generator=gen, device=device, dtype=torch.bfloat16)
            store.assign(b, np.arange(s0, s0 + m), k, v)
    cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
    return pool, store, cfg


def run_ours(args, rank, world, device):
    import torch
    import torch.distributed as dist

    from paper_2506_07311_b200 import _lib
    from paper_2506_07311_b200.attention import _Workspace
    from paper_2506_07311_b200.batch import DecodeBatch

    name, lengths, hq, hkv, d, ps = workload(args, rank, world)
    B = len(lengths)
    W, K = args.warmup, args.steps
    total_steps = W + K
    pool, store, cfg = build_cache(lengths, hq, hkv, d, ps, extra_tokens=2 * total_steps + 2,
                                   device=device, seed=rank)
    lib = _lib.load()
    # pre-grow capacity for every step (host allocator work stays out of `value`)
    for b, n in enumerate(lengths):
        pool.grow(b, n + total_steps)
    mirror = pool.device_table(device)
    rows_np = np.asarray([pool.table(b).mirror_row for b in range(B)], dtype=np.int32)
    base = np.asarray(lengths, dtype=np.int32)
    gen = torch.Generator(device=device).manual_seed(1234 + rank)
    qs = torch.randn((total_steps, B, hq, d), generator=gen, device=device, dtype=torch.bfloat16)
    ks = torch.randn((total_steps, B, hkv, d), generator=gen, device=device, dtype=torch.bfloat16)
    vs = torch.randn((total_steps, B, hkv, d), generator=gen, device=device, dtype=torch.bfloat16)
    # per-step metadata [q_seq | key counts | mirror rows | host work plan];
    # key counts grow by one per step (the appended token is attended)
    plans = [_lib.attention_plan(base + t + 1, rows_np, ps, hq, hkv, args.waves)
             for t in range(total_steps)]
    width = 3 * B + max(pl.size for pl in plans)
    meta_np = np.zeros((total_steps, width), dtype=np.int32)
    for t in range(total_steps):
        row_t = np.concatenate([np.arange(B, dtype=np.int32), base + t + 1, rows_np, plans[t]])
        meta_np[t, :row_t.size] = row_t
    meta = torch.from_numpy(meta_np).to(device)
    out = torch.empty((B, hq, d), dtype=torch.float32, device=device)
    ws_bytes = lib.pkv_attention_workspace_bytes(B, hq, d)
    ws = _Workspace.get(device, ws_bytes)
    l2_bytes = torch.cuda.get_device_properties(device).L2_cache_size
    # L2 flush between steps: *read* 2x L2 of unrelated data, so the next
    # step starts with a cold, clean L2 (a write flush would leave dirty lines
    # whose write-back steals HBM bandwidth from the timed kernel)
    flush_buf = torch.ones(max(2 * l2_bytes, 256 << 20) // 4, dtype=torch.float32, device=device)

    class _Flush:
        @staticmethod
        def zero_():
            flush_buf.sum()

    flush = _Flush()
    stream = torch.cuda.current_stream(device)
    sp = C.c_void_p(stream.cuda_stream)
    prof = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b_ in prof:  # materialise the underlying cudaEvent_t handles
        a.record(); b_.record()
    torch.cuda.synchronize(device)

    def make_args(t, prof_pair=None):
        # one decode step = K1 append fused into the K2 launch (the last split
        # of each sequence writes the new token into its page) + the split
        # combine (programmatic dependent launch) when a sequence is split
        mt = meta[t]
        md = mt.data_ptr()
        return _lib.AttentionArgs(
            q=qs[t].data_ptr(), q_dtype=_lib.PKV_BF16, n_queries=B, q_seq=md, q_nkeys=md + 4 * B,
            k_cache=store.keys.data_ptr(), v_cache=store.values.data_ptr(), kv_dtype=_lib.PKV_BF16,
            block_table=mirror.data_ptr(), bt_stride=mirror.shape[1], seq_row=md + 8 * B,
            seq_start=None, page_size=ps, hq=hq, hkv=hkv, head_dim=d, scale=cfg.scale,
            out=out.data_ptr(), out_dtype=_lib.PKV_F32, workspace=ws.data_ptr(),
            workspace_bytes=ws.numel(), num_sms=0, target_waves=args.waves,
            prof_start=prof_pair[0].cuda_event if prof_pair else None,
            prof_stop=prof_pair[1].cuda_event if prof_pair else None,
            mode=0, k_new=ks[t].data_ptr(), v_new=vs[t].data_ptr(),
            plan=md + 12 * B, plan_host=plans[t].ctypes.data)

    # argument blocks are built before the timed region so the host only
    # pays one C call per step (keeps host latency out of the device timing)
    step_args = [make_args(t, prof[t - W] if t >= W else None) for t in range(total_steps)]
    fn = lib.pkv_paged_attention

    def step(t, prof_pair=None):
        st = fn(C.byref(step_args[t]), sp)
        if st:
            _lib.check(st, "pkv_paged_attention")

    for t in range(W):
        flush.zero_()
        step(t)
    torch.cuda.synchronize(device)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)
    with ClockSampler(device.index) as clocks:
        for i in range(K):
            flush.zero_()  # L2 flush (untimed)
            starts[i].record(stream)
            step(W + i, prof[i])
            ends[i].record(stream)
        torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    k2_ms = [a.elapsed_time(b_) for a, b_ in prof]
    total_ms = sum(step_ms)
    # bytes of the steps actually timed (contexts grow by one token per step)
    alg_bytes = kv_bytes = 0
    for i in range(K):
        lens_t = [n + W + i + 1 for n in lengths]
        a_b, kv_b = algorithmic_bytes(lens_t, hq, hkv, d, ps)
        alg_bytes += a_b
        kv_bytes += kv_b
    tokens = B * K
    gathered = torch.tensor([total_ms, float(tokens), float(kv_bytes), float(alg_bytes), sum(k2_ms)],
                            dtype=torch.float64, device=device)
    if world > 1:
        tmax = gathered[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        sums = gathered[1:].clone()
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        total_ms_max = float(tmax.item())
        tokens_all, kv_all, alg_all = (float(x) for x in sums[:3].tolist())
    else:
        total_ms_max = total_ms
        tokens_all, kv_all, alg_all = float(tokens), float(kv_bytes), float(alg_bytes)

    result = {
        "name": name, "B": B, "step_ms": step_ms, "total_ms_max": total_ms_max,
        "tokens_all": tokens_all, "kv_all": kv_all, "alg_all": alg_all,
        "k2_ms_mean": sum(k2_ms) / K, "k2_alg_bytes_mean": alg_bytes / K,
        "clocks": clocks.summary(), "lengths": lengths, "shape": (hq, hkv, d, ps),
        # one decode launch per step (K1 append fused, split merge in-kernel)
        "launches": K,
    }
    if not args.no_e2e:
        result["e2e"] = run_e2e(args, pool, store, cfg, lengths, device, flush, world)
    return result


def run_e2e(args, pool, store, cfg, lengths, device, flush, world):
    """Same metric through the public API: DecodeBatch.step with pinned host
    q/k/v and a pinned host output (one native pkv_decode_step call per
    step); the H2D of the inputs and the D2H of the output are timed."""
    import torch
    import torch.distributed as dist

    from paper_2506_07311_b200.batch import DecodeBatch

    B = len(lengths)
    hq, hkv, d, ps = cfg.head_count, cfg.kv_head_count, cfg.head_dim, cfg.page_size
    batch = DecodeBatch(store, list(range(B)), cfg)
    W, K = max(2, args.warmup // 2), args.steps
    rng = np.random.default_rng(7)
    host = [(torch.from_numpy(rng.standard_normal((B, hq, d)).astype(np.float32)).bfloat16().pin_memory(),
             torch.from_numpy(rng.standard_normal((B, hkv, d)).astype(np.float32)).bfloat16().pin_memory(),
             torch.from_numpy(rng.standard_normal((B, hkv, d)).astype(np.float32)).bfloat16().pin_memory())
            for _ in range(4)]
    out_host = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()
    # pools were pre-grown for the device-timed phase; reset logical lengths
    # so every sequence continues from its current length
    lens0 = [pool.table(b).logical_len for b in range(B)]
    for b in range(B):
        pool.grow(b, lens0[b] + W + K + 1)
    times = []
    launches = 0
    h2d = d2h = 0
    for i in range(W + K):
        q, k, v = host[i % 4]
        flush.zero_()
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        # one native call: H2D q/k/v, allocator + plan, fused append +
        # decode (pkv_decode_step); the result crosses PCIe into the pinned
        # host output (stored by the kernel through the mapped pointer)
        batch.step(q, k, v, out=out_host)
        torch.cuda.current_stream(device).synchronize()
        dt = time.perf_counter() - t0
        if i >= W:
            times.append(dt)
            launches += batch.last_launches
            h2d += q.numel() * 2 + k.numel() * 2 + v.numel() * 2 + 4 * batch._stage.meta_used
            d2h += out_host.numel() * 4
    kv = 0
    for i in range(K):
        kv += sum(2 * (n + W + i + 1) * hkv * d * 2 for n in lens0)
    total = sum(times)
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
        kvt = torch.tensor([float(kv)], dtype=torch.float64, device=device)
        dist.all_reduce(kvt)
        kv = float(kvt.item())
    return {"value": kv / total / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d // K,
            "d2h_bytes_per_step": d2h // K, "ms_per_step": 1e3 * total / K,
            "tokens_per_s": B * K * world / total if world > 1 else B * K / total,
            "gpu_launches": launches}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port of the reference kernel on the host cores
# ---------------------------------------------------------------------------

def cpu_sample(args, lengths, hq, hkv, d, ps, budget_s=12.0, max_steps=None):
    """Time the oracle's restatement of the reference paged_attention
    (attention.py:259-354, GQA-folded when Hq != Hkv) on a sample of the
    workload's sequences; returns GB/s of algorithmic bf16-equivalent KV bytes
    and tokens/s.  fp32 values (bf16-rounded), as BASELINE.md §3 prescribes."""
    from oracle import OracleMeta, OraclePool, OracleStore
    from oracle.attention import fold_gqa_meta, fold_gqa_queries, round_bf16, streaming_attention
    from oracle.store import OracleBatchView

    # sample: every 4th sequence of the sorted workload (spans the length range)
    order = sorted(range(len(lengths)), key=lambda i: lengths[i])
    idx = order[::4] if len(lengths) >= 8 else order
    lens = [lengths[i] for i in idx]
    rng = np.random.default_rng(0)
    pool = OraclePool(sum(-(-(n + 1) // ps) for n in lens) + 2, ps)
    store = OracleStore(pool, hkv, d)
    for j, n in enumerate(lens):
        pool.reserve(j, n)
        store.assign(j, np.arange(n), round_bf16(rng.standard_normal((n, hkv, d)).astype(np.float32)),
                     round_bf16(rng.standard_normal((n, hkv, d)).astype(np.float32)))
    g = hq // hkv
    q = round_bf16(rng.standard_normal((len(lens), hq, d)).astype(np.float32))
    view = OracleBatchView(lens, ids=list(range(len(lens))))
    meta = fold_gqa_meta(OracleMeta.decode(view), g)
    rows = store.view_row_indices(view)
    qf = fold_gqa_queries(q, hkv)
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        # the reference gathers through the block table inside the kernel
        streaming_attention(qf, store.keys[rows], store.values[rows], meta,
                            scale=1.0 / math.sqrt(d), causal=True, tile=ps)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s or (max_steps and len(times) >= max_steps):
            break
    best = min(times)
    kv = sum(2 * n * hkv * d * 2 for n in lens)
    return {
        "value": kv / best / 1e9, "unit": "GB/s", "tokens_per_s": len(lens) / best,
        "cores": os.cpu_count(), "kind": "port",
        "sample": (f"{len(lens)} of {len(lengths)} sequences (every 4th by length, contexts "
                   f"{min(lens)}-{max(lens)}), oracle restatement of reference paged_attention, "
                   f"fp32 arithmetic on bf16-rounded values, numpy/OpenBLAS on all host threads, "
                   f"best of {len(times)} runs; bytes counted at bf16 size"),
        "ms_per_step": best * 1e3,
    }


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (oracle port) on the host."""
    name, lengths, hq, hkv, d, ps = workload(args, 0, 1)
    total = args.warmup + args.steps
    per_step = []
    res = None
    for i in range(total):
        res = cpu_sample(args, lengths, hq, hkv, d, ps, budget_s=0.0, max_steps=1)
        if i >= args.warmup:
            per_step.append(res["ms_per_step"])
    ms = statistics.mean(per_step)
    value = res["value"] * res["ms_per_step"] / ms
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
        "config": {"workload": name, "sample": res["sample"]},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": res["cores"], "kind": "port",
                         "sample": res["sample"]},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "tokens_per_s": res["tokens_per_s"] * res["ms_per_step"] / ms,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(config_name):
    """dram bytes per K2 launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        return s.get(config_name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    import __graft_entry__

    if rank == 0 and not os.path.exists(os.path.join(ROOT, "paper_2506_07311_b200", "libpkv200.so")):
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    r = run_ours(args, rank, world, device)
    if rank == 0:
        K = args.steps
        value = r["kv_all"] / (r["total_ms_max"] / 1e3) / 1e9
        peak, peak_src = load_peaks()
        k2_achieved = r["k2_alg_bytes_mean"] / (r["k2_ms_mean"] / 1e3) / 1e9
        traffic = load_traffic(args.config)
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": r["total_ms_max"] / K,
            "higher_is_better": True, "scaling": "strong" if args.config == "c5" else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (randn K/V/Q, scattered pages)",
            "config": {"workload": r["name"], "global_batch": int(r["tokens_all"] / K),
                       "kv_bytes_per_step": r["kv_all"] / K, "page_size": r["shape"][3],
                       "parallelism": f"request-sharded x{world}", "l2": "flushed between steps (read of 2x L2 of unrelated data)"},
            "pct_of_8TBs": round(100 * value / world / NOMINAL_HBM_GBS, 2),
            "tokens_per_s": r["tokens_all"] / (r["total_ms_max"] / 1e3),
            "roofline": {"bound": "hbm", "kernel": "decode_tc_kernel (K2-TC, K1 fused)", "achieved": round(k2_achieved, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(k2_achieved / peak, 4),
                         "traffic": traffic, "peak_source": peak_src,
                         "k2_ms_mean": r["k2_ms_mean"],
                         "k2_share_of_step": r["k2_ms_mean"] / (sum(r["step_ms"]) / K),
                         "algorithmic_bytes_per_launch": r["k2_alg_bytes_mean"]},
            "clocks": r["clocks"],
            "gpu_launches": r["launches"],
        }
        if "e2e" in r:
            e = r["e2e"]
            line["e2e"] = {"value": round(e["value"], 2), "unit": "GB/s",
                           "h2d_bytes_per_step": e["h2d_bytes_per_step"],
                           "d2h_bytes_per_step": e["d2h_bytes_per_step"],
                           "ms_per_step": e["ms_per_step"], "tokens_per_s": e["tokens_per_s"]}
        if world == 1 and not args.no_prefill:
            line["prefill_c4"] = prefill_c4(device)
        if world == 1 and not args.no_cpu_baseline:
            name, lengths, hq, hkv, d, ps = workload(args, 0, 1)
            cb = cpu_sample(args, lengths, hq, hkv, d, ps)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["cpu_baseline"]["tokens_per_s"] = cb["tokens_per_s"]
        print(json.dumps(line), flush=True)
        if args.sweep:
            sweep(device)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def prefill_c4(device, n=8192):
    """Side measurement of BASELINE.json configs[3] (C4): one 8192-token
    Llama-3-8B GQA prompt appended into the paged cache (K1) and attended
    causally by the K3 tcgen05 prefill kernel.  TFLOP/s under the reference
    FLOP convention 4*Hq*D*n(n+1)/2 (attention.py:224-226), CUDA events."""
    import torch

    from paper_2506_07311_b200 import AttentionConfig, KvStore, MaskMeta, PagePool, paged_attention

    hq, hkv, d, ps = 32, 8, 128, 16
    pool = PagePool(n // ps + 8, page_size=ps)
    store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=device)
    pool.reserve(0, n)
    g = torch.Generator(device=device).manual_seed(4)
    k = torch.randn((n, hkv, d), generator=g, device=device).bfloat16()
    v = torch.randn((n, hkv, d), generator=g, device=device).bfloat16()
    q = torch.randn((n, hq, d), generator=g, device=device).bfloat16()
    cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
    pos = np.arange(n)
    store.assign(0, pos, k, v)
    meta = MaskMeta.self_attention(store.batch_view([0]))
    from paper_2506_07311_b200.attention import _launch_prefill, suffix_runs

    runs = suffix_runs(meta)
    rows = np.asarray([pool.table(0).mirror_row], dtype=np.int32)
    mirror = pool.device_table(device)

    def kernel_only(ev):
        return _launch_prefill(q, meta, cfg, runs, k=store.keys, v=store.values, kv_code=store.dtype_code,
                               bt=mirror, rows=rows, out_dtype=torch.float32, device=device,
                               prof=(ev[0].cuda_event, ev[1].cuda_event) if ev else None)

    for _ in range(3):
        paged_attention(q, store, meta, cfg, precision="prefill")
        kernel_only(None)
    torch.cuda.synchronize(device)
    times, app, kern = [], [], []
    for _ in range(10):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        store.assign(0, pos, k, v)  # K1 over the whole prompt (host validation included)
        e1.record()
        paged_attention(q, store, meta, cfg, precision="prefill")
        e2.record()
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for x in ev:
            x.record()  # materialise the cudaEvent_t handles
        kernel_only(ev)
        torch.cuda.synchronize(device)
        app.append(e0.elapsed_time(e1))
        times.append(e1.elapsed_time(e2))
        kern.append(ev[0].elapsed_time(ev[1]))
    ms = sorted(times)[len(times) // 2]
    kms = sorted(kern)[len(kern) // 2]
    flops = 4 * hq * d * n * (n + 1) // 2
    tf = flops / (kms * 1e-3) / 1e12
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            sustained = float(json.load(f)["bf16_tflops_sustained"])
    except Exception:
        sustained = 1400.0
    return {"workload": f"C4 causal prefill, 1 x {n} tokens, GQA 32q/8kv x128 bf16, page 16",
            "kernel": "prefill_tc_kernel (K3, tcgen05/TMEM)", "kernel_ms": kms, "tflops": round(tf, 1),
            "frac_of_sustained_bf16": round(tf / sustained, 3), "api_ms": ms,
            "api_tflops": round(flops / (ms * 1e-3) / 1e12, 1), "append_ms": min(app),
            "note": "kernel_ms: CUDA events around the K3 launch; api_ms: the whole paged_attention() call "
                    "(host planning + metadata upload + launch); FLOPs per the reference convention"}


def sweep(device):
    """C3 context sweep (stderr): decode GB/s vs context at several batches."""
    import subprocess

    for ctx in (2048, 4096, 8192, 16384, 32768):
        for b in (1, 8, 64):
            if b * ctx * 4096 > 24 << 30:
                continue
            cmd = [sys.executable, os.path.abspath(__file__), "--config", "c3", "--context", str(ctx),
                   "--batch", str(b), "--steps", "10", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"]
            out = subprocess.run(cmd, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
            sys.stderr.write(f"SWEEP ctx={ctx} batch={b}: {line}\n")


if __name__ == "__main__":
    main()
